"""torchrun worker for multi-GPU executor parity (launched by
tests/test_executor_multigpu.py): every rank runs its stage of the plan and
checks its own layers' gradients / updated weights against the fp64 oracle."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from oracle.executor_ref import full_batch_step  # noqa: E402
from paper_2007_01045_b200.runtime import Executor, merge_timelines  # noqa: E402
from parity_util import check_grads, check_loss, check_update  # noqa: E402


def main():
    spec = json.loads(sys.argv[1])
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(rank)
    dist.init_process_group("gloo")
    model, plan, M, gbs = spec["model"], spec["plan"], spec["M"], spec["gbs"]
    sched = {"schedule": spec.get("schedule", "dapple"), "recompute": spec.get("recompute", False)}
    exact = full_batch_step(model, gbs)
    emu = full_batch_step(model, gbs, bf16=True)
    stage = next(s for s in plan["stages"] if rank in s["gpus"])
    layers = range(*stage["layers"])
    results = {}
    for apply in (False, True):
        ex = Executor(model, plan, M, gbs, lr=1e-3, rank=rank, world=world, apply=apply, **sched)
        loss = ex.step()
        if sched["schedule"] == "gpipe":
            # measured block order: every forward of this stage before its first backward
            blocks = [b for b in ex.timeline()["blocks"] if b[0] % 2 == 0 and b[3] >= 0]
            last_f = max(b[4] for b in blocks if b[2] == 0)
            first_b = min(b[3] for b in blocks if b[2] == 1)
            assert last_f <= first_b, (last_f, first_b)
        if stage is plan["stages"][-1]:
            check_loss(loss, emu, exact)
        if apply:
            results[apply] = check_update(ex, emu, layers, model["kind"], model, 1e-3)
        else:
            results[apply] = check_grads(ex, emu, exact, layers, model["kind"], model["layers"])
            if model.get("vocab"):
                from test_lm_gpu import _check_lm_tensors
                _check_lm_tensors(ex, emu, exact, stage is plan["stages"][0], stage is plan["stages"][-1])
        parts = [None] * world
        dist.all_gather_object(parts, ex.timeline())
        if rank == 0:
            tl = merge_timelines(parts, M, len(plan["stages"]))
            print(json.dumps({"plan": [[s["layers"], s["gpus"]] for s in plan["stages"]],
                              "latency_ms": tl["latency"] * 1e3, "bubble": tl["bubble"]}), flush=True)
        ex.close()
    # more steps must keep working (flag sequence numbers advance)
    ex = Executor(model, plan, M, gbs, lr=1e-3, rank=rank, world=world, **sched)
    ex.step()
    ex.step()
    ex.close()
    print(f"rank {rank} ok worst grad err {results[False]:.3g} weight err {results[True]:.3g}", flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
