"""Single-GPU executor parity: the full DAPPLE step (S=1 plan, M micro-batches
accumulated on the device) vs the fp64 CPU oracle on the same seed."""
import json

import numpy as np
import pytest

from oracle.executor_ref import full_batch_step
from parity_util import check_grads, check_loss, check_update

pytestmark = pytest.mark.gpu

CASES = [
    (dict(kind="mlp", layers=4, hidden=256), 32, 4),
    (dict(kind="mlp", layers=16, hidden=1024), 64, 8),  # C1 MLP16 at full size (configs[0])
    (dict(kind="bert", layers=2, hidden=256, heads=4, ffn=1024, seq=128), 8, 2),
    (dict(kind="gpt", layers=2, hidden=256, heads=4, ffn=1024, seq=128), 8, 4),
]


@pytest.mark.parametrize("model,gbs,M", CASES)
def test_single_gpu_step_matches_oracle(cuda, model, gbs, M):
    from paper_2007_01045_b200.runtime import Executor
    L = model["layers"]
    plan = {"stages": [{"layers": [0, L], "gpus": [0], "replication": 1}], "phi": [1]}
    exact = full_batch_step(model, gbs)
    emu = full_batch_step(model, gbs, bf16=True)
    ex = Executor(model, plan, M, gbs, lr=1e-3, apply=False)
    check_loss(ex.step(), emu, exact)
    check_grads(ex, emu, exact, range(L), model["kind"], L)
    ex.close()
    # and with the SGD apply: the fp32 master weights moved by -lr * grad
    ex = Executor(model, plan, M, gbs, lr=1e-3, apply=True)
    ex.step()
    check_update(ex, emu, range(L), model["kind"], model, 1e-3)
    ex.close()


def test_two_steps_loss_decreases(cuda):
    from paper_2007_01045_b200.runtime import Executor
    model = dict(kind="mlp", layers=4, hidden=256)
    plan = {"stages": [{"layers": [0, 4], "gpus": [0], "replication": 1}]}
    ex = Executor(model, plan, 4, 32, lr=0.5)
    l0 = ex.step()
    l1 = ex.step()
    l2 = ex.step()
    assert l2 < l1 < l0
    tl = ex.timeline()
    assert len(tl["blocks"]) == 2 * 4 and tl["step_s"] > 0
    ex.close()


@pytest.mark.parametrize("schedule,recompute", [("gpipe", False), ("dapple", True), ("gpipe", True)])
def test_single_gpu_schedules_match_oracle(cuda, schedule, recompute):
    """GPipe block order and re-computation leave the step's numerics unchanged."""
    from paper_2007_01045_b200.runtime import Executor
    model = dict(kind="bert", layers=2, hidden=256, heads=4, ffn=1024, seq=128)
    plan = {"stages": [{"layers": [0, 2], "gpus": [0], "replication": 1}]}
    exact = full_batch_step(model, 8)
    emu = full_batch_step(model, 8, bf16=True)
    ex = Executor(model, plan, 4, 8, lr=1e-3, apply=False, schedule=schedule, recompute=recompute)
    info = ex.info
    assert info["schedule"] == schedule and info["recompute"] == recompute
    assert info["stash_slots"] == (1 if recompute else 4 if schedule == "gpipe" else info["phi"])
    check_loss(ex.step(), emu, exact)
    check_grads(ex, emu, exact, range(2), "bert", 2)
    ex.close()


def test_layer_profiler_emits_reference_profile(cuda):
    """Executor.layer_profile: per-layer F/B measured on the GPU, in the
    reference's profile format (round-trips through load_profile)."""
    from paper_2007_01045_b200 import pipeplan
    from paper_2007_01045_b200.runtime import Executor
    model = dict(kind="bert", layers=3, hidden=256, heads=4, ffn=1024, seq=128)
    plan = {"stages": [{"layers": [0, 3], "gpus": [0], "replication": 1}]}
    ex = Executor(model, plan, 2, 8, apply=False)
    prof = ex.layer_profile(3)
    assert prof["profile_batch_size"] == 4
    assert len(prof["layers"]) == 3
    h = 256
    for l in prof["layers"]:
        assert l["fwd_time_us"] > 0 and l["bwd_time_us"] > l["fwd_time_us"] * 0.5
        assert l["activation_bytes"] == 4 * 128 * h * 2
        assert l["param_bytes"] == (12 * h * h + 13 * h) * 4
    loaded = pipeplan.call("load_profile", profile=json.dumps(prof))
    assert len(loaded["layers"]) == 3 and loaded["profile_batch_size"] == 4
    # the profiler leaves the gradient buffers clean: a step afterwards still matches the oracle
    exact = full_batch_step(model, 8)
    emu = full_batch_step(model, 8, bf16=True)
    check_loss(ex.step(), emu, exact)
    check_grads(ex, emu, exact, range(3), "bert", 3)
    ex.close()


def test_launch_count_covers_graph_replays(cuda):
    """Steps replay a captured CUDA graph; every replay adds the graph's kernel
    nodes to dpl_k_launch_count (captured launches themselves are not counted)."""
    from paper_2007_01045_b200 import _lib
    from paper_2007_01045_b200.runtime import Executor
    lib = _lib.lib()
    model = dict(kind="bert", layers=2, hidden=256, heads=4, ffn=1024, seq=128)
    plan = {"stages": [{"layers": [0, 2], "gpus": [0], "replication": 1}]}
    ex = Executor(model, plan, 2, 4)
    ex.step()  # capture + first replay
    c0 = lib.dpl_k_launch_count()
    ex.step()
    c1 = lib.dpl_k_launch_count()
    ex.step()
    c2 = lib.dpl_k_launch_count()
    ex.close()
    per_step = c1 - c0
    assert per_step > 50 and c2 - c1 == per_step
