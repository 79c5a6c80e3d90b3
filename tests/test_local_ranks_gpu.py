"""Multi-rank DAPPLE steps with every rank in this process on ONE GPU
(runtime.LocalRanks): the same per-rank step programs as one process per GPU
-- Split-Concat peer copies + flag waits between stages (N3 / N5), the
replica AllReduce over peer memory (N4, collective.cu), the per-rank chains
-- checked against the CPU oracle, so a 1-GPU box exercises the multi-rank
path.  The plans are the multi-GPU suite's (tests/test_executor_multigpu.py)."""
import json

import numpy as np
import pytest

from oracle.executor_ref import full_batch_step
from parity_util import check_grads, check_loss, check_update
from test_executor_multigpu import CASES, CASES8, SCHED_CASES

pytestmark = pytest.mark.gpu


def _run(model, plan, M, gbs, schedule="dapple", recompute=False):
    from paper_2007_01045_b200.runtime import LocalRanks, merge_timelines
    exact = full_batch_step(model, gbs)
    emu = full_batch_step(model, gbs, bf16=True)
    sched = dict(schedule=schedule, recompute=recompute)
    S = len(plan["stages"])
    for apply in (False, True):
        lr = LocalRanks(model, plan, M, gbs, lr=1e-3, apply=apply, **sched)
        try:
            losses = lr.step()
            for rank, ex in enumerate(lr.ranks):
                stage = next(s for s in plan["stages"] if rank in s["gpus"])
                layers = range(*stage["layers"])
                if stage is plan["stages"][-1]:
                    check_loss(losses[rank], emu, exact)
                if apply:
                    check_update(ex, emu, layers, model["kind"], model, 1e-3)
                else:
                    check_grads(ex, emu, exact, layers, model["kind"], model["layers"])
                    if model.get("vocab"):
                        from test_lm_gpu import _check_lm_tensors
                        _check_lm_tensors(ex, emu, exact, stage is plan["stages"][0], stage is plan["stages"][-1])
            # replicas of a stage hold bit-identical reduced gradients
            if not apply:
                for stage in plan["stages"]:
                    g = stage["gpus"]
                    l0 = stage["layers"][0]
                    name = "W" if model["kind"] in ("mlp", "vgg") else "W1"
                    n = emu.grads[(l0, name)].size
                    ref = lr.ranks[g[0]].read(l0, name, n, grad=True)
                    for r in g[1:]:
                        assert np.array_equal(lr.ranks[r].read(l0, name, n, grad=True), ref)
            tl = merge_timelines(lr.timelines(), M, S)
            assert tl["latency"] > 0 and 0.0 <= tl["bubble"] < 1.0
            # later steps keep working (flag banks alternate and are cleared)
            lr.step()
            lr.step()
        finally:
            lr.close()


@pytest.mark.parametrize("n,model,plan,M,gbs", [c for c in CASES if c not in CASES8])
def test_local_ranks_step_matches_oracle(cuda, n, model, plan, M, gbs):
    _run(model, plan, M, gbs)


@pytest.mark.parametrize("n,model,plan,M,gbs,schedule,recompute", SCHED_CASES)
def test_local_ranks_schedules_match_oracle(cuda, n, model, plan, M, gbs, schedule, recompute):
    _run(model, plan, M, gbs, schedule, recompute)


def test_local_ranks_measured_block_order(cuda):
    """The measured per-rank blocks follow the plan's chain: on every stage
    the forward of micro-batch i starts after its activations arrived (the
    previous stage's send ended) and backward i after the next stage's
    gradient send of i ended."""
    from paper_2007_01045_b200.runtime import LocalRanks, merge_timelines
    model = dict(kind="bert", layers=4, hidden=256, heads=4, ffn=1024, seq=128)
    plan = {"stages": [{"layers": [0, 2], "gpus": [0]}, {"layers": [2, 4], "gpus": [1]}], "phi": [2, 1]}
    M = 4
    lr = LocalRanks(model, plan, M, 8, apply=False)
    try:
        lr.step()
        tl = merge_timelines(lr.timelines(), M, 2)
    finally:
        lr.close()
    blk = {(x, i, k): (s, e) for x, i, k, s, e in tl["blocks"]}
    # the receiver is released by the flag store inside the send block, so its
    # block starts after the send started (the send's end event is recorded a
    # little after the flag store)
    eps = 2e-6  # event resolution
    for i in range(M):
        assert blk[(2, i, 0)][0] >= blk[(1, i, 0)][0] - eps  # F_i on stage 1 after its activation send began
        assert blk[(0, i, 1)][0] >= blk[(1, i, 1)][0] - eps  # B_i on stage 0 after its gradient send began
        assert blk[(1, i, 0)][0] >= blk[(0, i, 0)][1] - eps  # the send follows F_i on stage 0
        assert blk[(1, i, 1)][0] >= blk[(2, i, 1)][1] - eps  # the gradient send follows B_i on stage 1
    # stage 0 runs phi = 2 forwards before its first backward
    f = sorted((blk[(0, i, 0)][0], i) for i in range(M))
    b0 = blk[(0, 0, 1)][0]
    assert sum(1 for s, _ in f if s < b0) == 2


def test_local_ranks_info_reports_peer_allreduce(cuda):
    from paper_2007_01045_b200.runtime import LocalRanks
    model = dict(kind="mlp", layers=4, hidden=256)
    plan = {"stages": [{"layers": [0, 4], "gpus": [0, 1, 2]}]}
    lr = LocalRanks(model, plan, 2, 12, apply=False)
    try:
        lr.step()
        assert all(json.loads(json.dumps(ex.info))["replication"] == 3 for ex in lr.ranks)
        assert lr.ranks[0].allreduce == "peer"
    finally:
        lr.close()


@pytest.mark.parametrize("n,model,plan,M,gbs", CASES8, ids=["C2-2x4", "C4-8-stage"])
def test_local_ranks_eight_rank_plans(cuda, n, model, plan, M, gbs):
    """The 8-GPU plan shapes (C2: 2 stages x 4 replicas; C4: straight 8-stage
    LM pipeline) as eight ranks on one GPU: gradients, loss and the applied
    update vs the oracle, replicas bit-identical after the 4-way AllReduce."""
    _run(model, plan, M, gbs)
