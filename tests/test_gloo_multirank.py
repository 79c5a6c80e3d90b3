"""Host-side multi-rank logic under torch.distributed (gloo, world_size 2,
CPU): every rank derives the same Split-Concat routes and the same per-stage
chains from the plan, the timeline merge agrees across ranks, and the blob /
NCCL-id exchange protocol of runtime.Executor round-trips."""
import json
import os
import sys

import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _worker(rank, world, port, out_dir):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    import torch.distributed as dist
    from paper_2007_01045_b200 import pipeplan
    from paper_2007_01045_b200.runtime import merge_timelines
    dist.init_process_group("gloo", rank=rank, world_size=world)
    plan = {"stages": [{"layers": [0, 3], "gpus": [0]}, {"layers": [3, 4], "gpus": [1]}], "phi": [2, 1]}
    mine = {
        "routes": pipeplan.call("splitconcat_routes", plan=plan, boundary=0, micro_batch=6, rows_per_sample=4)["routes"],
        "chain": pipeplan.stage_chain(4, pipeplan.expand_plan_phi(plan["phi"])[2 * rank]),
    }
    allv = [None] * world
    dist.all_gather_object(allv, mine)
    assert allv[0]["routes"] == allv[1]["routes"]
    # synthetic per-rank measured blocks: stage 0 F then B, stage 1 later
    blocks = [[2 * rank, i, k, 0.1 * i + rank + k, 0.1 * i + rank + k + 0.05] for i in range(4) for k in (0, 1)]
    tl = {"t0_ns": 1_000_000_000 + rank * 1000, "step_s": 3.0, "blocks": blocks}
    parts = [None] * world
    dist.all_gather_object(parts, tl)
    merged = merge_timelines(parts, 4, 2)
    blobs = [None] * world
    dist.all_gather_object(blobs, bytes([rank]) * 64)
    assert b"".join(blobs) == bytes([0]) * 64 + bytes([1]) * 64
    with open(os.path.join(out_dir, f"r{rank}.json"), "w") as f:
        json.dump({"chain": mine["chain"], "latency": merged["latency"], "bubble": merged["bubble"]}, f)
    dist.destroy_process_group()


def test_two_rank_host_logic(tmp_path):
    mp.spawn(_worker, args=(2, 29533, str(tmp_path)), nprocs=2, join=True)
    r0 = json.load(open(tmp_path / "r0.json"))
    r1 = json.load(open(tmp_path / "r1.json"))
    assert r0["latency"] == pytest.approx(r1["latency"]) and r0["bubble"] == pytest.approx(r1["bubble"])
    assert [c[0] for c in r0["chain"]] == ["F", "F", "B", "F", "B", "F", "B", "B"]
    assert [c[0] for c in r1["chain"]] == ["F", "B"] * 4
