"""Step parity at the BASELINE.json shapes (full width, reduced depth / batch
so the CPU oracle finishes in seconds to a minute):

  C2  BERT-48 layer shape: h 1024, seq 512, 16 heads, FFN 4096
  C4  GPT-2 1.5B layer shape: h 1600, seq 1024, 25 heads, FFN 6400, V 50257
      (LM ends included; vocabulary not a multiple of 8)
  C3  VGG-19 at 224 x 224 (64..512 channels, FC 4096, 1000 classes)
  C1  MLP16 h 1024 on the planner's S=2 plan, phi [3,1], GBS 64, M 8

against the bf16-emulating oracle (oracle/executor_ref.py, fp64 arithmetic,
bf16 rounding where the device stores bf16).  Stated tolerance: every
gradient tensor within 2% relative Frobenius error, loss within 0.2%.

VGG is teacher-forced: a 1-ulp bf16 difference in a conv output can move a
2x2 pool maximum and reroute a gradient, and such flips compound over 16
convs, so each layer is re-run by the oracle on the device's own stashed
input / pre-pool output / output gradient (Executor probes) and its weight,
bias and input gradients must agree within 2% -- a real dgrad / wgrad bug in
any layer fails this regardless of depth (measured worst 0.26%); the loss
must agree within 0.2% and the free-running whole-step gradients are only
sanity-bounded.  The transformer shapes are checked both ways."""
import numpy as np
import pytest

from oracle.executor_ref import Model, bf16_round, full_batch_step, init_layer, layer_backward, layer_forward
from parity_util import rel_fro, tensor_names

pytestmark = pytest.mark.gpu

TOL = 0.02
LOSS_TOL = 2e-3

C2 = dict(kind="bert", layers=2, hidden=1024, heads=16, ffn=4096, seq=512)
C4 = dict(kind="gpt", layers=2, hidden=1600, heads=25, ffn=6400, seq=1024, vocab=50257)
C3 = dict(kind="vgg", layers=19, image=224, width=64, fc=4096, classes=1000)
C1 = dict(kind="mlp", layers=16, hidden=1024)


def _check_step(ranks, plan, model, emu, loss, tol=TOL):
    """Loss and every gradient of every rank vs the bf16 oracle."""
    assert abs(loss - emu.loss) <= LOSS_TOL * abs(emu.loss), (loss, emu.loss)
    worst = 0.0
    for rank, ex in enumerate(ranks):
        stage = next(s for s in plan["stages"] if rank in s["gpus"])
        for l in range(*stage["layers"]):
            for name in tensor_names(model["kind"]):
                want = emu.grads[(l, name)]
                e = rel_fro(ex.read(l, name, want.size, grad=True), want)
                assert e < tol, f"rank {rank} layer {l} {name}: {e:.4g}"
                worst = max(worst, e)
        if model.get("vocab"):
            first, last = stage is plan["stages"][0], stage is plan["stages"][-1]
            names = ([("emb", "wte"), ("emb", "wpe")] if first else []) + \
                ([("head", "Wout"), ("head", "lnf_g"), ("head", "lnf_b")] if last else [])
            for owner, name in names:
                want = emu.grads[(owner, name)]
                e = rel_fro(ex.read(owner, name, want.size, grad=True), want)
                assert e < tol, f"rank {rank} {owner}.{name}: {e:.4g}"
                worst = max(worst, e)
    return worst


def _last_loss(losses):
    return [l for l in losses if l == l][-1]


@pytest.mark.parametrize("model,gbs,M", [(C2, 8, 4), (C4, 2, 2)], ids=["C2", "C4"])
def test_single_gpu_step_at_baseline_width(cuda, model, gbs, M):
    from paper_2007_01045_b200.runtime import Executor
    plan = {"stages": [{"layers": [0, 2], "gpus": [0], "replication": 1}]}
    emu = full_batch_step(model, gbs, bf16=True)
    ex = Executor(model, plan, M, gbs, apply=False)
    try:
        _check_step([ex], plan, model, emu, ex.step())
    finally:
        ex.close()


@pytest.mark.parametrize("model,plan,gbs,M", [
    # C2's shape: 2 stages x 2 replicas, 2-sample replica slices (as at GBS 64, M 8, r 4)
    (C2, {"stages": [{"layers": [0, 1], "gpus": [0, 1]}, {"layers": [1, 2], "gpus": [2, 3]}]}, 8, 2),
    # C4's shape: a straight pipeline with the embedding / LM head on the end stages
    (C4, {"stages": [{"layers": [0, 1], "gpus": [0]}, {"layers": [1, 2], "gpus": [1]}]}, 2, 2),
], ids=["C2-2x2", "C4-straight"])
def test_pipelined_step_at_baseline_width_on_one_gpu(cuda, model, plan, gbs, M):
    from paper_2007_01045_b200.runtime import LocalRanks
    emu = full_batch_step(model, gbs, bf16=True)
    lr = LocalRanks(model, plan, M, gbs, apply=False)
    try:
        _check_step(lr.ranks, plan, model, emu, _last_loss(lr.step()))
    finally:
        lr.close()


def _teacher_forced(ex, model, layers, samples, tol=TOL):
    """Each layer re-run by the oracle on the device's own input and output
    gradient (M = 1, so the device's accumulated gradients are this one
    micro-batch's)."""
    from oracle.executor_ref import elems_per_sample, vgg_layer
    m = Model.from_dict(model)
    worst = {}
    for l in layers:
        nx, ny = samples * elems_per_sample(m, l), samples * elems_per_sample(m, l + 1)
        x = ex.probe(l, "x", nx)
        y = ex.probe(l, "y", ny)
        dy = ex.probe(l, "dy", ny)
        p = {k: v.astype(np.float64) for k, v in init_layer(m, l, 1234).items()}
        rows = x.reshape(samples * (m.seq if m.kind != "vgg" else 1), -1)
        y_o, cache = layer_forward(m, l, p, rows, samples, q=bf16_round)
        e_y = rel_fro(y, y_o)
        assert e_y < 0.01, f"layer {l} forward: {e_y:.4g}"
        if m.kind == "vgg":
            v = vgg_layer(m, l)
            # the backward routes through the device's own pre-pool output
            post = ex.probe(l, "aux", samples * v["h"] * v["w"] * v["cout"]) if v.get("pool") else y
            cache = (rows, post.reshape(-1, v["cout"]) if v["conv"] else post.reshape(samples, -1))
        dx_o, g = layer_backward(m, l, p, cache, dy.reshape(y_o.shape), samples, need_dx=l > 0, q=bf16_round)
        for name in tensor_names(m.kind):
            got = ex.read(l, name, g[name].size, grad=True)
            e = rel_fro(got, g[name])
            assert e < tol, f"layer {l} d{name} (teacher-forced): {e:.4g}"
            worst[(l, name)] = e
        if l > 0:
            e = rel_fro(ex.probe(l, "dx", nx), dx_o)
            assert e < tol, f"layer {l} dx (teacher-forced): {e:.4g}"
            worst[(l, "dx")] = e
    return worst


def test_vgg19_224_teacher_forced_and_step(cuda):
    """C3: VGG-19 at 224 x 224, 2 samples, one micro-batch."""
    from paper_2007_01045_b200.runtime import Executor
    plan = {"stages": [{"layers": [0, 19], "gpus": [0], "replication": 1}]}
    ex = Executor(C3, plan, 1, 2, apply=False, probe=True)
    try:
        loss = ex.step()
        worst = _teacher_forced(ex, C3, range(19), 2)
        print("teacher-forced worst", max(worst.values()))
        assert max(worst.values()) < TOL
        emu = full_batch_step(C3, 2, bf16=True)
        assert abs(loss - emu.loss) <= LOSS_TOL * abs(emu.loss), (loss, emu.loss)
        # Whole-step gradients vs the free-running oracle: the pool-argmax /
        # ReLU flips of 16 convs reach the classifier's inputs (measured ~12%
        # on FC1's weight gradient at 224 x 224), so this is only a sanity
        # bound -- the per-layer teacher-forced check above is the criterion.
        for l in (16, 17, 18):
            for name in ("W", "b"):
                want = emu.grads[(l, name)]
                assert rel_fro(ex.read(l, name, want.size, grad=True), want) < 0.3
    finally:
        ex.close()


@pytest.mark.parametrize("model", [C2, C4], ids=["C2", "C4"])
def test_transformer_layers_teacher_forced(cuda, model):
    from paper_2007_01045_b200.runtime import Executor
    plan = {"stages": [{"layers": [0, 2], "gpus": [0], "replication": 1}]}
    ex = Executor(model, plan, 1, 1, apply=False, probe=True)
    try:
        ex.step()
        _teacher_forced(ex, model, range(2), 1)
    finally:
        ex.close()


def test_c1_planner_plan_executes_on_one_gpu(cuda):
    """C1 exactly: the host planner picks [0,9)x1 [9,16)x1 with phi [3,1] for
    MLP16 (SURVEY §8(d) recipe: 20 / 40 us per layer, seps [2], 0.35 GiB per
    GPU); that plan runs as two ranks on one GPU (Split-Concat hand-off and
    flag chain included) at GBS 64, M 8, and matches both the scheduled CPU
    restatement of the same plan and the full-batch oracle."""
    import json
    from oracle.executor_ref import scheduled_step
    from paper_2007_01045_b200 import pipeplan
    from paper_2007_01045_b200.runtime import LocalRanks
    h = 1024
    prof = {"profile_batch_size": 64, "layers": [
        {"fwd_time_us": 20.0, "bwd_time_us": 40.0, "activation_bytes": 8 * h * 4, "param_bytes": (h * h + h) * 4}
        for _ in range(16)]}
    cluster = {"seps": [2], "intra_bw_gbps": 770.0, "inter_bw_gbps": 50.0, "intra_latency_us": 5.0,
               "inter_latency_us": 10.0, "per_gpu_memory_gb": 0.35}
    plan = pipeplan.plan(prof, cluster, 8)["plan"]
    assert [s["layers"] for s in plan["stages"]] == [[0, 9], [9, 16]], json.dumps(plan)
    assert plan["phi"] == [3, 1]
    emu = full_batch_step(C1, 64, bf16=True)
    sched = scheduled_step(C1, plan, 8, 64)
    exact = full_batch_step(C1, 64)
    # the CPU restatement of the scheduled step is the full-batch step (fp64)
    for key in exact.grads:
        assert rel_fro(sched.grads[key], exact.grads[key]) < 1e-10
    lr = LocalRanks(C1, plan, 8, 64, apply=False)
    try:
        loss = _last_loss(lr.step())
        assert lr.ranks[0].info["phi"] == 3 and lr.ranks[1].info["phi"] == 1
        # ReLU chain: bf16 rounding flips grow toward the input (parity_util)
        for rank, ex in enumerate(lr.ranks):
            stage = plan["stages"][rank]
            for l in range(*stage["layers"]):
                tol = TOL + 0.004 * (15 - l)
                for name in ("W", "b"):
                    want = emu.grads[(l, name)]
                    e = rel_fro(ex.read(l, name, want.size, grad=True), want)
                    assert e < tol, f"layer {l} {name}: {e:.4g}"
        assert abs(loss - emu.loss) <= LOSS_TOL * abs(emu.loss)
        assert abs(loss - sched.loss) <= 1e-2 * abs(sched.loss)
    finally:
        lr.close()
