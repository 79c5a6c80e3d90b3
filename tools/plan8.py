"""The planner's self-consistent plan choice for N = 2 / 4 / 8 B200s of one
node, from layer profiles measured on THIS GPU (bench.plan_fixed_point: the
reference planner's plan() plus its top-k runners-up, each priced with
simulate_plan on profiles at its own replica slice sizes).  Planning needs
no more GPUs than one; this is the plan bench.py would run at N = 8.

    python tools/plan8.py [--model bert48] [--mem-gb 12]
"""
import argparse
import json
import sys
import time

sys.path.insert(0, ".")
import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="bert48")
    ap.add_argument("--mem-gb", type=float, default=None)
    ap.add_argument("--gpus", type=int, nargs="+", default=[2, 4, 8])
    args = ap.parse_args()
    model = bench.MODELS[args.model]
    dflt = bench.DEFAULTS.get(args.model, {})
    m = dflt.get("micro_batches", 8)
    gbs = dflt.get("global_batch") or 64
    mb = gbs // m
    mem = args.mem_gb if args.mem_gb is not None else (12.0 if args.model == "bert48" else 180.0)
    profiles = {mb: bench.profile_model(model, mb)}
    out = []
    for n in args.gpus:
        t0 = time.time()
        plan, info = bench.plan_fixed_point(model, profiles, mb, bench.b200_cluster(n, mem), m)
        step_ms = info["sim_latency_ms"]
        out.append({"n_gpus": n, "plan": [[s["layers"], s["gpus"]] for s in plan["stages"]], "phi": plan.get("phi"),
                    "planner_sim_ms": step_ms, "predicted_samples_per_s": gbs / step_ms * 1e3,
                    "candidates": info["candidates"], "plan_s": time.time() - t0})
        print(json.dumps(out[-1]))
    return out


if __name__ == "__main__":
    main()
