"""Runs one multi-rank plan with every rank in this process on cuda:0
(runtime.LocalRanks) and prints the per-rank losses and step times.
    python tools/local_probe.py [mlp2|mlp_dp|bert2] [steps]"""
import json
import sys
import time

sys.path.insert(0, ".")
from paper_2007_01045_b200.runtime import LocalRanks  # noqa: E402

CASES = {
    "mlp2": (dict(kind="mlp", layers=4, hidden=256),
             {"stages": [{"layers": [0, 2], "gpus": [0]}, {"layers": [2, 4], "gpus": [1]}]}, 4, 24),
    "mlp_dp": (dict(kind="mlp", layers=4, hidden=256), {"stages": [{"layers": [0, 4], "gpus": [0, 1]}]}, 4, 24),
    "bert2": (dict(kind="bert", layers=4, hidden=256, heads=4, ffn=1024, seq=128),
              {"stages": [{"layers": [0, 1], "gpus": [0]}, {"layers": [1, 4], "gpus": [1]}]}, 4, 8),
    "mlp31": (dict(kind="mlp", layers=4, hidden=256),
              {"stages": [{"layers": [0, 3], "gpus": [0, 1, 2]}, {"layers": [3, 4], "gpus": [3]}]}, 4, 24),
    "mlp13": (dict(kind="mlp", layers=4, hidden=256),
              {"stages": [{"layers": [0, 1], "gpus": [0]}, {"layers": [1, 4], "gpus": [1, 2, 3]}]}, 4, 24),
    "mlp_dp3": (dict(kind="mlp", layers=4, hidden=256), {"stages": [{"layers": [0, 4], "gpus": [0, 1, 2]}]}, 4, 24),
    "mlp_22": (dict(kind="mlp", layers=4, hidden=256),
               {"stages": [{"layers": [0, 2], "gpus": [0, 1]}, {"layers": [2, 4], "gpus": [2, 3]}]}, 4, 24),
}
import faulthandler  # noqa: E402
faulthandler.dump_traceback_later(40, exit=True)
name = sys.argv[1] if len(sys.argv) > 1 else "mlp2"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
model, plan, M, gbs = CASES[name]
print("building", name, flush=True)
lr = LocalRanks(model, plan, M, gbs, apply=False)
print("connected", flush=True)
for k in range(steps):
    t = time.perf_counter()
    for r, ex in enumerate(lr.ranks):
        ex.step_launch()
        print(f"  launched rank {r}", flush=True)
    losses = []
    for r, ex in enumerate(lr.ranks):
        losses.append(ex.step_finish())
        print(f"  finished rank {r}", flush=True)
    print(json.dumps({"step": k, "losses": losses, "s": time.perf_counter() - t}), flush=True)
lr.close()
print("ok", flush=True)
