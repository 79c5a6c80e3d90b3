"""Profiles a model's layers on one B200 (Executor.layer_profile -> the
reference's profile JSON) and runs the host planner (pipeplan.plan, bit-exact
with the reference) for G GPUs under a few per-GPU memory caps.

    python tools/profile_plan.py --model bert48 --mb 8 16 32 --out gpurun_out/profiles
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from bench import MODELS  # noqa: E402


def profile(model, mb, reps):
    from paper_2007_01045_b200.runtime import Executor
    L = model["layers"]
    plan = {"stages": [{"layers": [0, L], "gpus": [0], "replication": 1}]}
    ex = Executor(model, plan, 1, mb, rank=0, world=1, device=0, timeline=False)
    prof = ex.layer_profile(reps)
    ex.close()
    return prof


def cluster(g, mem_gb):
    return {"seps": [g], "intra_bw_gbps": 770.0, "inter_bw_gbps": 50.0, "intra_latency_us": 5.0,
            "inter_latency_us": 10.0, "per_gpu_memory_gb": mem_gb}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="bert48")
    ap.add_argument("--mb", type=int, nargs="+", default=[8])
    ap.add_argument("--M", type=int, default=8)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--gpus", type=int, nargs="+", default=[2, 4, 8])
    ap.add_argument("--mem", type=float, nargs="+", default=[180.0, 20.0, 10.0, 5.0])
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    import torch
    torch.cuda.set_device(0)
    from paper_2007_01045_b200 import pipeplan
    model = MODELS[args.model]
    for mb in args.mb:
        prof = profile(model, mb, args.reps)
        f = sum(l["fwd_time_us"] for l in prof["layers"])
        b = sum(l["bwd_time_us"] for l in prof["layers"])
        print(json.dumps({"model": args.model, "mb": mb, "fwd_ms": f / 1e3, "bwd_ms": b / 1e3,
                          "layer0": prof["layers"][0], "layer_last": prof["layers"][-1]}), flush=True)
        if args.out:
            os.makedirs(args.out, exist_ok=True)
            with open(os.path.join(args.out, f"profile_{args.model}_mb{mb}.json"), "w") as fh:
                json.dump(prof, fh, indent=1)
        for g in args.gpus:
            for mem in args.mem:
                try:
                    p = pipeplan.plan(prof, cluster(g, mem), args.M)["plan"]
                    sim = pipeplan.simulate_plan(p, prof, cluster(g, mem), args.M)
                    print(json.dumps({"mb": mb, "G": g, "mem_gb": mem,
                                      "plan": [[s["layers"], s["gpus"]] for s in p["stages"]],
                                      "phi": p.get("phi"), "sim_ms": sim["latency"] * 1e3}), flush=True)
                except Exception as e:  # infeasible under the cap
                    print(json.dumps({"mb": mb, "G": g, "mem_gb": mem, "error": str(e)[:120]}), flush=True)


if __name__ == "__main__":
    main()
