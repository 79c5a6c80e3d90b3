"""Generates tests/golden/planner_golden.json by running the *reference*
pipeplan library (oracle/_ref/ref_cli, built from /root/reference/proj/src by
oracle/Makefile) on a fixed corpus: the reference's own unit-test cases,
random plan / brute-force / simulate instances, and the BASELINE planner
sweeps (C5: AmoebaNet-36 / XLNet-36 synthetic profiles at G = 1/2/4/8, and a
BERT-48 profile on an 8-GPU NVSwitch node).  The fixtures let the GPU box
(no /root/reference there) check bit-exact planner parity.

    python tests/golden/make_golden.py
"""
import json
import os
import random
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.refproc import ReferenceProcess  # noqa: E402


def seq(fwd, bwd, ar=None):
    return [{"kind": "compute", "fwd": f, "bwd": b, "allreduce": (ar[i] if ar else 0.0)}
            for i, (f, b) in enumerate(zip(fwd, bwd))]


def cluster(seps, intra=100.0, inter=10.0, lat_in=1.0, lat_out=10.0, mem=16.0):
    return {"seps": seps, "intra_bw_gbps": intra, "inter_bw_gbps": inter, "intra_latency_us": lat_in,
            "inter_latency_us": lat_out, "per_gpu_memory_gb": mem}


def uniform_profile(n, f=1000.0, b=2000.0, act=0, params=0):
    return {"profile_batch_size": 1, "layers": [{"fwd_time_us": f, "bwd_time_us": b, "activation_bytes": act,
                                                 "param_bytes": params} for _ in range(n)]}


def xlnet36():
    # uniform transformer blocks (Table I shape): equal compute and weights
    return {"profile_batch_size": 8, "layers": [
        {"fwd_time_us": 4200.0, "bwd_time_us": 8600.0, "activation_bytes": 8 << 20, "param_bytes": 50 << 20}
        for _ in range(36)]}


def amoebanet36():
    # conv cells: activations shrink and parameters grow with depth
    layers = []
    for i in range(36):
        stage = i // 12
        layers.append({"fwd_time_us": 2600.0 + 150.0 * (i % 12), "bwd_time_us": 5300.0 + 310.0 * (i % 12),
                       "activation_bytes": (96 >> stage) << 20, "param_bytes": (2 << stage) << 20})
    return {"profile_batch_size": 8, "layers": layers}


def bert48_b200():
    # per-layer F/B of a 64-sample micro-batch on one B200 (measured by bench.py, round 1)
    return {"profile_batch_size": 64, "layers": [
        {"fwd_time_us": 2410.0, "bwd_time_us": 7300.0, "activation_bytes": 64 * 512 * 1024 * 2,
         "param_bytes": 12596224 * 4} for _ in range(48)]}


def corpus():
    rng = random.Random(2007_01045)
    reqs = []
    # simulator_test.cpp / estimator_test.cpp hand cases
    reqs += [{"op": "schedule", "seq": seq([1.5], [2.25]), "M": 1, "phi": [1]},
             {"op": "schedule", "seq": seq([1, 1], [1, 1]), "M": 2, "phi": [2, 1]},
             {"op": "schedule", "seq": seq([1, 1], [1, 1]), "M": 2, "schedule": "gpipe"},
             {"op": "schedule", "seq": seq([1] * 4, [2] * 4), "M": 7, "phi": [4, 3, 2, 1]},
             {"op": "schedule", "seq": seq([1] * 4, [2] * 4), "M": 7, "schedule": "gpipe"},
             {"op": "schedule", "seq": seq([0.3, 0.7, 0.2], [0.9, 0.4, 0.6]), "M": 6, "phi": [3, 2, 1]},
             {"op": "schedule", "seq": seq([1] * 3, [1] * 3), "M": 4, "phi": [3, 2]},
             {"op": "schedule", "seq": seq([1] * 3, [1] * 3), "M": 4, "phi": [2, 3, 1]},
             {"op": "estimate", "seq": seq([1.5], [2.5]), "M": 1},
             {"op": "estimate", "seq": seq([1] * 4, [2] * 4), "M": 7},
             {"op": "estimate", "seq": seq([1, 3, 1], [2, 6, 2]), "M": 4},
             {"op": "estimate", "seq": seq([3, 1, 1], [6, 2, 2]), "M": 4},
             {"op": "estimate", "seq": seq([2 / 3, 10 / 3, 1], [4 / 3, 20 / 3, 2]), "M": 4},
             {"op": "optimize_phi", "seq": seq([1] * 5, [2] * 5), "M": 16, "phi_strategy": "preset_a", "D": 16},
             {"op": "optimize_phi", "seq": seq([1] * 5, [2] * 5), "M": 16, "phi_strategy": "preset_b", "D": 16},
             {"op": "optimize_phi", "seq": seq([1] * 5, [2] * 5), "M": 16, "phi_strategy": "preset_a", "D": 3},
             {"op": "optimize_phi", "seq": seq([1] * 5, [2] * 5), "M": 2, "phi_strategy": "preset_b", "D": 16},
             {"op": "optimize_phi", "seq": seq([1] * 5, [2] * 5), "M": 4, "phi_strategy": "preset_a", "D": 0},
             {"op": "expand_plan_phi", "phi": [3, 2, 1]},
             {"op": "expand_plan_phi", "phi": []},
             {"op": "allreduce_time", "size": 1000000000, "devices": [0, 1], "cluster": cluster([2], 100, 10, 0, 0)},
             {"op": "allreduce_time", "size": 0, "devices": [1, 2], "cluster": cluster([2, 2], 100, 10, 0, 1000)},
             {"op": "allreduce_time", "size": 1000000000, "devices": [0, 2], "cluster": cluster([2])},
             {"op": "allreduce_time", "size": 1000000000, "devices": [], "cluster": cluster([2])},
             {"op": "splitconcat_time", "size": 1000000000, "src": [0], "dst": [1], "cluster": cluster([1, 1], 100, 10, 0, 0)},
             {"op": "splitconcat_time", "size": 1000000000, "src": [0], "dst": [8, 9], "cluster": cluster([8, 8], 100, 10, 0, 2)},
             {"op": "splitconcat_time", "size": 1000000000, "src": [0, 1], "dst": [1, 0], "cluster": cluster([2, 2])},
             {"op": "splitconcat_time", "size": 0, "src": [0], "dst": [2], "cluster": cluster([2, 2], 100, 10, 3, 7)},
             {"op": "enumerate_placements", "cluster": cluster([8, 8]), "count": 8},
             {"op": "enumerate_placements", "cluster": cluster([8, 8]), "count": 4, "free": [4, 8]},
             {"op": "enumerate_placements", "cluster": cluster([8, 8]), "count": 2},
             {"op": "enumerate_placements", "cluster": cluster([8, 8]), "count": 3, "free": [2, 5]},
             {"op": "enumerate_placements", "cluster": cluster([8, 8]), "count": 17},
             {"op": "memory_feasible", "param_bytes": 100, "act": 50, "injected": 1, "capacity": 850},
             {"op": "memory_feasible", "param_bytes": 100, "act": 50, "injected": 2, "capacity": 850},
             {"op": "memory_feasible", "param_bytes": 100, "act": 50, "injected": 1, "capacity": 0},
             {"op": "plan", "profile": uniform_profile(16), "cluster": cluster([8, 8], 100, 10, 0, 0), "M": 16},
             {"op": "plan", "profile": uniform_profile(16, 3000, 6000, 4 << 20, 60 << 20),
              "cluster": cluster([8, 8], 130, 3.125, 1, 10), "M": 16},
             {"op": "plan", "profile": uniform_profile(1), "cluster": cluster([1, 1, 1]), "M": 4},
             {"op": "plan", "profile": uniform_profile(2, 1000, 2000, 0, 1 << 20), "cluster": cluster([1, 1], mem=1e-7),
              "M": 4},
             {"op": "plan", "profile": uniform_profile(5, 1200, 2400, 1 << 20, 4 << 20),
              "cluster": cluster([1, 1, 1], 20, 20, 1, 1), "M": 6, "top_k": 4, "report": True},
             {"op": "load_profile", "profile": '{"profile_batch_size": 4, "layers": [{"fwd_time_us": 1000, '
                                               '"bwd_time_us": 2000, "activation_bytes": 10, "param_bytes": 20}]}'},
             {"op": "load_profile", "profile": '{"profile_batch_size": 4, "layers": [{"fwd_time_us": 1000, '
                                               '"bwd_time_us": 2000, "activation_bytes": 1.5, "param_bytes": 20}]}'},
             {"op": "load_profile", "profile": '{"profile_batch_size": 4, "layers": []}'},
             {"op": "load_cluster", "cluster": cluster([8, 8], 130, 3.125, 1, 10, 16)},
             {"op": "load_cluster", "cluster": cluster([], 130, 3.125, 1, 10, 16)},
             {"op": "load_cluster", "cluster": cluster([8], 0, 3.125, 1, 10, 16)}]
    # acceptance.cpp criterion 7 shapes
    vgg = {"profile_batch_size": 1, "layers": [
        {"fwd_time_us": f, "bwd_time_us": 2 * f, "activation_bytes": a << 20, "param_bytes": p << 20}
        for f, a, p in zip([8000] * 7 + [2000], [64, 48, 32, 24, 16, 8, 3, 1], [4] * 7 + [400])]}
    reqs.append({"op": "plan", "profile": vgg, "cluster": cluster([1, 1, 1, 1], 1.25, 1.25, 10, 10), "M": 16})
    reqs.append({"op": "plan", "profile": uniform_profile(16, 3000, 6000, 4 << 20, 60 << 20),
                 "cluster": cluster([8, 8], 130, 3.125, 1, 10), "M": 32})
    # BASELINE C5 planner sweep + BERT-48 on one 8xB200 node (NVSwitch: seps [G])
    nv = lambda g, mem: cluster([g], 770, 50, 5, 10, mem)  # noqa: E731
    for name, prof in (("xlnet36", xlnet36()), ("amoebanet36", amoebanet36())):
        for g in (1, 2, 4, 8):
            for strat in ("preset_a", "preset_b"):
                reqs.append({"op": "plan", "profile": prof, "cluster": nv(g, 180.0), "M": 16, "phi_strategy": strat,
                             "tag": f"C5 {name} G={g}"})
            reqs.append({"op": "plan", "profile": prof, "cluster": nv(g, 2.0), "M": 16, "tag": f"C5 {name} G={g} 2GiB"})
    for mem in (180.0, 5.0, 3.0):
        reqs.append({"op": "plan", "profile": bert48_b200(), "cluster": nv(8, mem), "M": 8, "tag": f"C2 bert48 {mem}GiB"})
    # random differential instances (planner, brute force, simulate)
    for _ in range(60):
        n = rng.randint(1, 12)
        prof = {"profile_batch_size": 1, "layers": [{"fwd_time_us": rng.uniform(100, 5000),
                                                     "bwd_time_us": rng.uniform(200, 9000),
                                                     "activation_bytes": rng.randint(0, 8 << 20),
                                                     "param_bytes": rng.randint(0, 64 << 20)} for _ in range(n)]}
        cl = cluster(rng.choice([[1], [2], [4], [8], [2, 2], [4, 4], [1, 3], [3, 3, 2]]), rng.choice([50, 130, 770]),
                     rng.choice([3.125, 12.5]), 1, 10, rng.choice([0.5, 2, 16]))
        M = rng.randint(1, 16)
        strat = rng.choice(["preset_a", "preset_b", "search"])
        reqs.append({"op": "plan", "profile": prof, "cluster": cl, "M": M, "phi_strategy": strat})
        if sum(cl["seps"]) <= 4 and n <= 8:
            reqs.append({"op": "brute_force_plan", "profile": prof, "cluster": cl, "M": M, "phi_strategy": strat})
        s = rng.randint(1, 6)
        sq = seq([rng.uniform(0.05, 2) for _ in range(s)], [rng.uniform(0.05, 2) for _ in range(s)],
                 [rng.uniform(0, 1) for _ in range(s)])
        m = rng.randint(1, 12)
        phi = [1] * s
        for x in range(s - 2, -1, -1):
            phi[x] = rng.randint(phi[x + 1], min(m, phi[x + 1] + 3))
        reqs.append({"op": "schedule", "seq": sq, "M": m, "phi": phi})
        reqs.append({"op": "schedule", "seq": sq, "M": m, "schedule": "gpipe"})
        reqs.append({"op": "estimate", "seq": sq, "M": m})
        reqs.append({"op": "optimize_phi", "seq": sq, "M": m, "phi_strategy": "search", "D": m})
    return reqs


def main():
    ref = ReferenceProcess()
    out = []
    plans = []
    for r in corpus():
        resp = ref.call(r)
        out.append({"request": r, "response": resp})
        if r["op"] in ("plan", "brute_force_plan") and "plan" in resp:
            plans.append((r, resp["plan"]))
    # simulate every produced plan under both schedules (+ recompute)
    for r, p in plans[:80]:
        for sched, rc in (("dapple", False), ("gpipe", False), ("dapple", True)):
            q = {"op": "simulate_plan", "plan": p, "profile": r["profile"], "cluster": r["cluster"], "M": r["M"],
                 "schedule": sched, "recompute": rc}
            out.append({"request": q, "response": ref.call(q)})
    ref.close()
    path = os.path.join(HERE, "planner_golden.json")
    with open(path, "w") as f:
        json.dump(out, f, separators=(",", ":"))
    print(f"{len(out)} cases -> {path} ({os.path.getsize(path) / 1e6:.1f} MB)")


if __name__ == "__main__":
    main()
