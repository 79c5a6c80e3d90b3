"""Host planner wall time, sequential vs parallel (DPL_PLANNER_THREADS), on
synthetic profiles; checks the plans are identical."""
import json
import os
import random
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def prof(n, seed=1):
    r = random.Random(seed)
    return {"profile_batch_size": 8, "layers": [
        {"fwd_time_us": r.uniform(100, 1000), "bwd_time_us": r.uniform(200, 2000),
         "activation_bytes": r.randint(1 << 20, 1 << 26), "param_bytes": r.randint(1 << 20, 1 << 27)}
        for _ in range(n)]}


def run(n, seps, threads):
    code = f"""
import json, sys, time; sys.path.insert(0, {ROOT!r})
from paper_2007_01045_b200 import pipeplan
from tools.planner_speed import prof
cl = {{"seps": {seps}, "intra_bw_gbps": 770.0, "inter_bw_gbps": 50.0, "intra_latency_us": 5.0,
      "inter_latency_us": 10.0, "per_gpu_memory_gb": 80.0}}
t = time.time(); p = pipeplan.plan(prof({n}), cl, 16, report=True); dt = time.time() - t
print(json.dumps({{"s": dt, "plan": p["plan"], "states": p["report"]["states_evaluated"]}}))
"""
    env = dict(os.environ, DPL_PLANNER_THREADS=str(threads))
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, check=True).stdout
    return json.loads(out.strip().splitlines()[-1])


if __name__ == "__main__":
    cases = [(36, [8]), (48, [8]), (24, [8, 8])]
    for n, seps in cases:
        a = run(n, seps, 1)
        b = run(n, seps, os.cpu_count())
        print(json.dumps({"layers": n, "seps": seps, "states": a["states"], "seq_s": round(a["s"], 3),
                          "par_s": round(b["s"], 3), "threads": os.cpu_count(), "speedup": round(a["s"] / b["s"], 2),
                          "identical": a["plan"] == b["plan"]}), flush=True)
