#!/usr/bin/env python
"""bench.py -- DAPPLE synchronous pipelined-DP training step on B200.

Workload (BASELINE.json configs[1], C2): BERT-48 encoder, hidden 1024, seq
512, 16 heads, FFN 4096, bf16, MSE regression head, synthetic data, global
batch 64 at every N (strong scaling), M = 8 micro-batches of 8 samples.  Plans:
  N = 1   [0,48) x1                         (the step: 8 micro-batches accumulated)
  N >= 2  the host planner's plan (bit-exact to the reference planner) on
          B200 layer profiles taken at the plan's own replica slice sizes,
          per_gpu_memory_gb 12 so that pure DP is infeasible (C2: 2 stages x
          4 replicas at N = 8, 2-sample replica slices).
--model gpt2-1.5b (configs[3], C4): GPT-2 1.5B with token embedding and
causal-LM cross-entropy head (vocab 50257), a straight N-stage pipeline,
M = 32 micro-batches of 1 sample (GBS 32 at every N: strong scaling).

Metric: training samples/s of the whole job (value: device-timed, inputs
generated in HBM; e2e: through the public API with pinned host inputs /
targets copied in and the loss read back every step), plus the measured
pipeline bubble and the planner-predicted vs measured batch latency L.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl dapple|reference]
  torchrun --nproc-per-node N bench.py --gpus N ...
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

MODELS = {
    "bert48": dict(kind="bert", layers=48, hidden=1024, heads=16, ffn=4096, seq=512),
    # C4: GPT-2 1.5B, causal-LM cross-entropy over the 50257-token vocabulary (projection stored padded to 50264 rows, padding masked)
    "gpt2-1.5b": dict(kind="gpt", layers=48, hidden=1600, heads=25, ffn=6400, seq=1024, vocab=50257),
    "mlp16": dict(kind="mlp", layers=16, hidden=1024),
    # C5's XLNet-36 (Table I: 36 uniform transformer blocks) executed as
    # a BERT-style encoder of that depth; its plans come from the host planner
    # on this model's own B200 profile (--plan planner), measured L vs est / sim L
    "xlnet36": dict(kind="bert", layers=36, hidden=1024, heads=16, ffn=4096, seq=512),
    # C5's AmoebaNet-36 (Table I: 36 conv cells in 3 resolution
    # stages, activations shrinking and parameters growing with depth) as a
    # 36-layer conv net of the VGG family: 12 + 12 + 11 3x3 convs at widths
    # 128 / 256 / 512 with a 2x2 pool after each stage, then the classifier
    "amoebanet36": dict(kind="vgg", layers=36, image=128, width=128, fc=4096, classes=1000,
                        convs=[12, 12, 11], mults=[1, 2, 4], fcs=1),
    # C3: VGG-19 on 224x224 images, 1000-class cross-entropy (convs as im2col + tcgen05 GEMM)
    "vgg19": dict(kind="vgg", layers=19, image=224, width=64, fc=4096, classes=1000),
}
METRIC = "training samples/sec at 1/2/4/8 B200; pipeline bubble %; predicted-vs-measured L"
PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


def vgg_shapes(m: dict) -> list:
    """The conv net's profile layers (csrc/runtime/layers.cu vgg_layer):
    VGG-19 by default, or the groups / multipliers / FC count given."""
    out, hw, cin = [], m["image"], 3
    for convs, mult in zip(m.get("convs", (2, 2, 4, 4, 4)), m.get("mults", (1, 2, 4, 8, 8))):
        for c in range(convs):
            cout = m["width"] * mult
            out.append(dict(conv=True, h=hw, w=hw, cin=cin, cout=cout, pool=c == convs - 1))
            cin = cout
        hw //= 2
    fcs = m.get("fcs", 3)
    for f in range(fcs):
        out.append(dict(conv=False, fin=hw * hw * cin if f == 0 else m["fc"],
                        fout=m["classes"] if f == fcs - 1 else m["fc"]))
    return out


def flops_per_sample(m: dict) -> float:
    """GEMM + attention-matmul FLOPs of one sample, fwd + dgrad + wgrad
    (24h^2 + 4sh per token per layer, x3)."""
    if m["kind"] == "mlp":
        return 6.0 * m["hidden"] ** 2 * m["layers"]
    if m["kind"] == "vgg":  # 19.634 GMAC fwd at 224 x 224, x2 x3
        f = 0.0
        for v in vgg_shapes(m):
            f += 2.0 * v["h"] * v["w"] * 9 * v["cin"] * v["cout"] if v["conv"] else 2.0 * v["fin"] * v["fout"]
        return 3.0 * f
    h, s, f = m["hidden"], m["seq"], m["ffn"]
    per_token = 2 * (4 * h * h + 2 * h * f) + 4 * s * h
    head = 2.0 * h * m.get("vocab", 0)  # LM head projection (SURVEY: 160,822,400 FLOP/token at V=50257)
    return 3.0 * (per_token * m["layers"] + head) * s


# per-workload defaults (BASELINE.json configs): C2 BERT-48 2 stages x N/2,
# M=8; C4 GPT-2 a straight N-stage pipeline, M=32 micro-batches of 1 sample
DEFAULTS = {"bert48": dict(micro_batches=8, slice=8, straight=False, global_batch=64),
            "gpt2-1.5b": dict(micro_batches=32, slice=1, straight=True),
            "mlp16": dict(micro_batches=8, slice=8, straight=False),
            "xlnet36": dict(micro_batches=16, slice=8, straight=False, global_batch=128),
            "amoebanet36": dict(micro_batches=16, slice=8, straight=False, global_batch=128),
            "vgg19": dict(micro_batches=8, slice=24, straight=False)}


def plan_fixed_point(model: dict, profiles: dict, mb: int, cluster: dict, m: int, max_iter: int = 5):
    """The host planner's plan (pipeplan.plan, bit-exact to the reference's
    planner.cpp:306-421) on B200 layer profiles taken at the plan's OWN
    replica slice sizes.  The reference cost model divides a stage's time by
    r (model.cpp:228-230), i.e. assumes perfect strong scaling of a layer over
    smaller slices, so: profile at mb and plan; profile every layer at the
    slice its stage runs (times x r, slice_profile) and evaluate the plan on
    that, its own profile (simulate_plan, planner.cpp:491-514); re-plan on
    it; stop when the planner proposes a plan already evaluated.  Among the
    proposals the one with the lowest self-consistent simulated L is run; its
    est / sim L are the planner's model evaluated at the times its replicas
    actually run at."""
    from paper_2007_01045_b200 import pipeplan

    def key(pl):
        return json.dumps([[s["layers"], s["gpus"]] for s in pl["stages"]])

    cands = {}
    history = []
    # Start from the full micro-batch profile and, so the choice does not hinge
    # on which proposals one chain happens to visit, also from the profile at
    # the slice of every replication factor r <= the GPU count (a plan whose
    # stages run r-way replicas is priced at the time they really take).
    n_gpus = sum(cluster.get("seps", [1]))
    starts = [mb] + sorted({-(-mb // r) for r in range(2, n_gpus + 1)} - {mb}, reverse=True)
    fixed = False
    for start in starts:
        if start not in profiles:
            profiles[start] = profile_model(model, start)
        prof = profiles[start]
        chain = []
        def evaluate(pl):
            k = key(pl)
            if k not in cands:
                for st in pl["stages"]:
                    size = -(-mb // len(st["gpus"]))
                    if size not in profiles:
                        profiles[size] = profile_model(model, size)
                own = slice_profile(profiles, pl, mb)
                seq = pipeplan.build_stage_sequence(pl, own, cluster)
                est = pipeplan.estimate_latency(seq, m)["total"]
                sim = pipeplan.simulate_plan(pl, own, cluster, m)["latency"]
                cands[k] = (pl, own, est, sim)
            return k

        for _ in range(max_iter):
            rep = pipeplan.plan(prof, cluster, m, report=True)
            res = rep["plan"]
            k = key(res)
            seen = k in cands
            evaluate(res)
            # the planner's runners-up (its top-k) are priced on their own
            # slice profiles too: which plan wins on the self-consistent
            # profile should not hinge on profile noise steering the chain
            for alt in (rep.get("report") or {}).get("top", []):
                evaluate(alt["plan"])
            chain.append({"start_slice": start, "stages": json.loads(k), "phi": res.get("phi"),
                          "planner_est_ms": res.get("est_latency_us", 0) / 1e3,
                          "planner_sim_ms": res.get("sim_latency_us", 0) / 1e3,
                          "own_profile_est_ms": cands[k][2] * 1e3, "own_profile_sim_ms": cands[k][3] * 1e3})
            if seen:
                break
            prof = cands[k][1]
        if start == mb:
            fixed = len(chain) >= 2 and chain[-1]["stages"] == chain[-2]["stages"]
        history += chain
    best = min(cands.values(), key=lambda c: c[3])
    plan, own, est, sim = best
    visited = {json.dumps(it["stages"]) for it in history}
    alternatives = [{"stages": json.loads(k), "own_profile_est_ms": c[2] * 1e3, "own_profile_sim_ms": c[3] * 1e3}
                    for k, c in cands.items() if k not in visited]
    return plan, {"iterations": history, "alternatives": alternatives, "fixed_point": fixed,
                  "candidates": len(cands),
                  "per_gpu_memory_gb": cluster["per_gpu_memory_gb"],
                  "est_latency_ms": est * 1e3, "sim_latency_ms": sim * 1e3,
                  "profile": "B200 layer profiles at the plan's own replica slice sizes"}


def make_plan(n: int, layers: int, straight: bool = False, kind: str = "", conv_layers: int = 16) -> dict:
    if n == 1:
        return {"stages": [{"layers": [0, layers], "gpus": [0], "replication": 1}]}
    if kind == "vgg":  # C3: conv stage on N - N/4 GPUs, FC stage on N/4 (6 + 2 at N = 8)
        fc = max(1, n // 4)
        return {"stages": [{"layers": [0, conv_layers], "gpus": list(range(n - fc)), "replication": n - fc},
                           {"layers": [conv_layers, layers], "gpus": list(range(n - fc, n)), "replication": fc}]}
    if straight:
        cuts = [layers * k // n for k in range(n + 1)]
        return {"stages": [{"layers": [cuts[k], cuts[k + 1]], "gpus": [k], "replication": 1} for k in range(n)]}
    half = n // 2
    cut = layers // 2
    return {"stages": [{"layers": [0, cut], "gpus": list(range(half)), "replication": half},
                       {"layers": [cut, layers], "gpus": list(range(half, n)), "replication": n - half}]}


def load_peaks() -> tuple[dict, str]:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except Exception:
        return PEAKS_FALLBACK, "fallback"


class ClockSampler:
    """SM clocks / throttle reasons sampled during the timed region: NVML
    polled every 5 ms from a thread (a short timed region -- VGG-19 at N=4 is
    ~100 ms -- still gets samples), nvidia-smi -lms 200 where NVML is absent."""
    # nvmlClocksEventReason* bits
    NVML_BITS = {"sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40}

    def _nvml_start(self) -> bool:
        try:
            import pynvml
            pynvml.nvmlInit()
            handles = [pynvml.nvmlDeviceGetHandleByIndex(i) for i in range(pynvml.nvmlDeviceGetCount())]
            reasons_fn = getattr(pynvml, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                pynvml.nvmlDeviceGetCurrentClocksThrottleReasons
            smax = [pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM) for h in handles]
        except Exception:
            return False
        self.nvml = True
        self.stop_evt = threading.Event()

        def poll():
            while not self.stop_evt.is_set():
                ts = time.time()
                for h, cmax in zip(handles, smax):
                    try:
                        clk = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                        power = pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0
                        bits = reasons_fn(h)
                    except Exception:
                        continue
                    order = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
                    flags = ["Active" if bits & self.NVML_BITS[n] else "Not Active" for n in order]
                    self.lines.append((ts, ", ".join(["", "", str(clk), str(cmax), str(power)] + flags)))
                self.stop_evt.wait(0.005)

        self.thread = threading.Thread(target=poll, daemon=True)
        self.thread.start()
        return True
    FIELDS = ["timestamp", "index", "clocks.sm", "clocks.max.sm", "power.draw", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap"]

    def __init__(self):
        self.proc = None
        self.nvml = False
        self.lines = []

    def start(self):
        if self._nvml_start():
            return
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "--query-gpu=" + ",".join(self.FIELDS),
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.time(), line.strip()))

    def mark(self, name):
        setattr(self, name, time.time())

    def stop(self) -> dict:
        if self.nvml:
            self.stop_evt.set()
            self.thread.join(timeout=5)
        elif not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        else:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        sm, smax, reasons, n_all = [], [], set(), 0
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        t0, t1 = getattr(self, "t_start", 0.0), getattr(self, "t_stop", float("inf"))
        for ts, line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < len(self.FIELDS) or not (t0 <= ts <= t1):
                continue
            try:
                clk, cmax, power = float(parts[2]), float(parts[3]), float(parts[4])
            except ValueError:
                continue
            n_all += 1
            for name, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(name)
            if power >= 250.0:  # under load (idle B200 draws ~150 W)
                sm.append(clk)
                smax.append(cmax)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples_under_load": len(sm), "samples": n_all,
                "source": "nvml 5 ms" if self.nvml else "nvidia-smi 200 ms"}


def dist_setup():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo")
    return rank, world


def gather(obj, world):
    if world == 1:
        return [obj]
    import torch.distributed as dist
    out = [None] * world
    dist.all_gather_object(out, obj)
    return out


def broadcast(obj, world):
    if world == 1:
        return obj
    import torch.distributed as dist
    box = [obj]
    dist.broadcast_object_list(box, src=0)
    return box[0]


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def host_batches(model: dict, plan: dict, rank: int, m: int, B: int, seed: int):
    """Pinned host copies of this rank's input / target slices of every
    micro-batch (the e2e leg's H2D sources): generated once by the library's
    own device generator (dpl_k_fill_uniform_bf16, the same keyed hash the
    executor uses), then copied to pinned host memory before timing."""
    import torch
    from paper_2007_01045_b200 import kernels
    stages = plan["stages"]
    k = next(i for i, s in enumerate(stages) if rank in s["gpus"])
    rep = stages[k]["gpus"].index(rank)
    r = len(stages[k]["gpus"])
    s0, s1 = B * rep // r, B * (rep + 1) // r  # this replica's samples of each micro-batch
    seq, h = model.get("seq", 1), model.get("hidden", 0)
    rows = (s1 - s0) * seq

    vocab = model.get("vocab", 0)
    if model["kind"] == "vgg":  # images [M][samples * H*W*3] bf16, labels [M][samples] int32
        e0 = model["image"] ** 2 * 3
        n = s1 - s0
        inp = tgt = None
        if k == 0:
            x = torch.empty((m, n * e0), dtype=torch.bfloat16, device="cuda")
            for i in range(m):
                kernels.fill_uniform_bf16(x[i], n * e0, seed, 1, (i * B + s0) * e0)
            torch.cuda.synchronize()
            inp = x.cpu().pin_memory()
        if k == len(stages) - 1:
            lab = torch.empty((m, n), dtype=torch.int32, device="cuda")
            for i in range(m):
                kernels.fill_tokens(lab[i], n, seed, 2, i * B + s0, model["classes"])
            torch.cuda.synchronize()
            tgt = lab.cpu().pin_memory()
        return inp, tgt

    def gen(tensor_id):
        if vocab:  # token ids [M][rows] int32
            out = torch.empty((m, rows), dtype=torch.int32, device="cuda")
            for i in range(m):
                kernels.fill_tokens(out[i], rows, seed, tensor_id, (i * B + s0) * seq, vocab)
        else:
            out = torch.empty((m, rows, h), dtype=torch.bfloat16, device="cuda")
            for i in range(m):
                kernels.fill_uniform_bf16(out[i], rows * h, seed, tensor_id, (i * B + s0) * seq * h)
        torch.cuda.synchronize()
        return out.cpu().pin_memory()

    inp = gen(1) if k == 0 else None            # tensor ids of layers.h kTensorInput / kTensorTarget
    tgt = gen(2) if k == len(stages) - 1 else None
    return inp, tgt


def b200_cluster(n: int, mem_gb: float = 180.0, link: dict | None = None) -> dict:
    """ClusterSpec of one NVSwitch node (model.cpp:175-199 units).  intra_bw /
    intra_latency come from this run's peer-copy sweep (calibrate_link) when
    there is a second GPU, else the recipe's measured 770 GB/s peer copy
    (B200_PROFILING.md); inter_* is unused on one node but must be > 0."""
    bw, lat = (link["bw_gbps"], link["latency_us"]) if link else (770.0, 5.0)
    return {"seps": [n], "intra_bw_gbps": bw, "inter_bw_gbps": 50.0, "intra_latency_us": lat,
            "inter_latency_us": 10.0, "per_gpu_memory_gb": mem_gb}


def calibrate_link(reps: int = 20) -> dict:
    """Peer copies cuda:0 -> cuda:1 over NVLink (copy engines, the path the
    Split-Concat hand-off takes) at 256 KiB .. 64 MiB, timed with CUDA events;
    least-squares fit t = latency + bytes / bw (costmodel.cpp:52-71's flow
    model).  Rank 0 only, before the executors exist."""
    import torch
    sizes = [1 << 18, 1 << 20, 1 << 22, 1 << 24, 1 << 26]
    src = torch.empty(sizes[-1], dtype=torch.uint8, device="cuda:0")
    dst = torch.empty(sizes[-1], dtype=torch.uint8, device="cuda:1")
    pts = []
    for n in sizes:
        for _ in range(3):
            dst[:n].copy_(src[:n], non_blocking=True)
        torch.cuda.synchronize(0)
        torch.cuda.synchronize(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            dst[:n].copy_(src[:n], non_blocking=True)
        b.record()
        b.synchronize()
        pts.append((n, a.elapsed_time(b) * 1e-3 / reps))
    xs = [n for n, _ in pts]
    ys = [t for _, t in pts]
    mx, my = statistics.mean(xs), statistics.mean(ys)
    slope = sum((x - mx) * (y - my) for x, y in zip(xs, ys)) / sum((x - mx) ** 2 for x in xs)
    lat = max(my - slope * mx, 0.0)
    return {"bw_gbps": 1.0 / slope / 1e9, "latency_us": lat * 1e6,
            "points": [{"bytes": n, "us": t * 1e6, "gbps": n / t / 1e9} for n, t in pts],
            "how": "cuda:0 -> cuda:1 tensor copies (cudaMemcpyPeerAsync, copy engines), CUDA events, "
                   f"{reps} back to back per size; fit t = latency + bytes / bw"}


def profile_model(model: dict, mb: int, reps: int = 5) -> dict:
    """The B200 layer profile (reference profile JSON, model.cpp:162-173):
    every layer's F/B timed on this GPU at the micro-batch size, in step order
    (Executor.layer_profile)."""
    from paper_2007_01045_b200.runtime import Executor
    L = model["layers"]
    ex = Executor(model, {"stages": [{"layers": [0, L], "gpus": [0], "replication": 1}]}, 1, mb,
                  rank=0, world=1, timeline=False, apply=False)
    try:
        return ex.layer_profile(reps)
    finally:
        ex.close()


def slice_profile(profiles: dict, plan: dict, mb: int) -> dict:
    """The executed plan's profile at the sizes its replicas actually run:
    stage k's layers take the layer times profiled at the largest replica
    slice ceil(mb / r_k), scaled by r_k so aggregate_stage's division by r
    (model.cpp:228-229) returns the slice time."""
    base = profiles[mb]
    layers = [dict(l) for l in base["layers"]]
    for st in plan["stages"]:
        r = len(st["gpus"])
        sl = profiles[-(-mb // r)]
        for l in range(*st["layers"]):
            layers[l]["fwd_time_us"] = sl["layers"][l]["fwd_time_us"] * r
            layers[l]["bwd_time_us"] = sl["layers"][l]["bwd_time_us"] * r
    return {**base, "layers": layers}


def calibrated_profile(model, plan, timelines, base=None) -> dict:
    """Per-layer F/B of the full micro-batch from a run's measured blocks
    (block time x r / layers on the stage)."""
    stages = plan["stages"]
    per_layer = {}
    for k, st in enumerate(stages):
        f_times, b_times = [], []
        for tl in timelines:
            if tl["stage"] != k:
                continue
            for x, i, kind, s, e in tl["blocks"]:
                if x == 2 * k and s >= 0:
                    (f_times if kind == 0 else b_times).append(e - s)
        lo, hi = st["layers"]
        r = len(st["gpus"])
        f = statistics.median(f_times) * r / (hi - lo)
        b = statistics.median(b_times) * r / (hi - lo)
        for l in range(lo, hi):
            per_layer[l] = (f, b)
    if base is not None:  # byte counts from the B200 profiler's profile
        return {**base, "layers": [{**base["layers"][l], "fwd_time_us": per_layer[l][0] * 1e6,
                                    "bwd_time_us": per_layer[l][1] * 1e6} for l in range(model["layers"])]}
    h = model["hidden"]
    params = (12 * h * h + 13 * h) * 4 if model["kind"] != "mlp" else (h * h + h) * 4
    return {"profile_batch_size": 8, "layers": [
        {"fwd_time_us": per_layer[l][0] * 1e6, "bwd_time_us": per_layer[l][1] * 1e6,
         "activation_bytes": 8 * model.get("seq", 1) * h * 2, "param_bytes": params} for l in range(model["layers"])]}


def predicted_latency(plan, profile, cluster, m, n, schedule="dapple"):
    """est_latency (estimator.cpp:56-86) and sim_latency (simulate_plan,
    planner.cpp:491-514) of the executed plan under `profile`, plus the
    simulated bubble."""
    from paper_2007_01045_b200 import pipeplan
    stages = plan["stages"]
    seq = pipeplan.build_stage_sequence(plan, profile, cluster)
    est = pipeplan.estimate_latency(seq, m)
    # the measured B blocks already contain any re-computed forward, so a
    # calibrated profile is simulated without apply_recompute
    sim = pipeplan.simulate_plan(plan, profile, cluster, m, schedule=schedule)
    busy = 0.0
    for x, i, kind, s, e in sim["timeline"]["blocks"]:
        if x % 2 == 0:
            busy += (e - s) * len(stages[x // 2]["gpus"])
    return {"est_ms": est["total"] * 1e3, "sim_ms": sim["latency"] * 1e3,
            "sim_bubble": 1.0 - busy / (n * sim["latency"]), "pivot": est["pivot"]}


def planner_cpu_times(profile: dict, cluster: dict, m: int, plan_json: dict) -> dict:
    """the reference's own plan() and
    simulate_plan() (oracle/_ref/ref_cli, compiled from /root/reference) on
    this run's profile and cluster, timed on this host beside the new host
    planner (sequential and parallel search) for the same request; the plans
    must be identical."""
    from oracle import refproc  # checker / CPU baseline only
    req = {"op": "plan", "profile": profile, "cluster": cluster, "M": m}
    sim = {"op": "simulate_plan", "plan": plan_json, "profile": profile, "cluster": cluster, "M": m}
    out = {"cores": os.cpu_count(), "M": m, "layers": len(profile["layers"]), "gpus": cluster["seps"]}
    from paper_2007_01045_b200 import pipeplan
    t = time.perf_counter()
    mine = pipeplan.call("plan", profile=profile, cluster=cluster, M=m, threads=1)
    out["ours_plan_seq_s"] = time.perf_counter() - t
    t = time.perf_counter()
    mine_par = pipeplan.call("plan", profile=profile, cluster=cluster, M=m, threads=os.cpu_count())
    out["ours_plan_par_s"] = time.perf_counter() - t
    t = time.perf_counter()
    mine_sim = pipeplan.simulate_plan(plan_json, profile, cluster, m)
    out["ours_simulate_s"] = time.perf_counter() - t
    if not refproc.available():
        out["reference"] = "oracle/_ref/ref_cli not built (needs /root/reference at build time)"
        return out
    ref = refproc.ReferenceProcess()
    try:
        t = time.perf_counter()
        theirs = ref.call(req)
        out["reference_plan_s"] = time.perf_counter() - t
        t = time.perf_counter()
        theirs_sim = ref.call(sim)
        out["reference_simulate_s"] = time.perf_counter() - t
    finally:
        ref.close()
    out["identical_plan"] = theirs.get("plan") == mine.get("plan") == mine_par.get("plan")
    out["identical_sim_latency"] = theirs_sim.get("latency") == mine_sim.get("latency")
    return out


def comm_stats(tls: list, link: dict | None) -> dict:
    """Split-Concat and replica-AllReduce traffic of one measured step (every
    rank's timeline): bytes moved and the achieved rate against the link.
    Split-Concat: each send block moves send_bytes (forward) / send_back_bytes
    (backward) from one rank.  AllReduce: bus bandwidth 2(r-1)/r x bytes / t
    per parameter block (the ring formula costmodel.cpp:41-50 charges)."""
    link_bw = link["bw_gbps"] if link else 770.0
    sc_bytes, sc_rates, sc_time = 0, [], 0.0
    ar_bytes, ar_rates, ar_time, impl = 0, [], 0.0, "none"
    for tl in tls:
        x0 = 2 * tl["stage"]
        for x, i, kind, st, en in tl["blocks"]:
            if x == x0 or st < 0 or en <= st:
                continue
            nbytes = tl.get("send_bytes", 0) if kind == 0 else tl.get("send_back_bytes", 0)
            if nbytes:
                sc_bytes += nbytes
                sc_time += en - st
                sc_rates.append(nbytes / (en - st) / 1e9)
        r = tl.get("replication", 1)
        for blk, st, en, nbytes in tl.get("allreduce", []):
            if en > st and r > 1:
                impl = tl.get("allreduce_impl", impl)
                ar_bytes += nbytes
                ar_time += en - st
                ar_rates.append(2.0 * (r - 1) / r * nbytes / (en - st) / 1e9)
    out = {"link_gbps": link_bw, "link_source": "this run's peer-copy fit" if link else "B200_PROFILING.md 770 GB/s"}
    if sc_rates:
        med = statistics.median(sc_rates)
        out["splitconcat"] = {"bytes_per_step": sc_bytes, "sends": len(sc_rates), "gbps_median": med,
                              "gbps_aggregate": sc_bytes / sc_time / 1e9, "frac_of_link": med / link_bw,
                              "frac_of_nvlink_nominal": med / 900.0}
    if ar_rates:
        med = statistics.median(ar_rates)
        out["allreduce"] = {"impl": impl, "bytes_per_step": ar_bytes, "blocks": len(ar_rates),
                            "busbw_gbps_median": med, "busbw_gbps_aggregate": sum(ar_rates) / len(ar_rates),
                            "frac_of_link": med / link_bw, "frac_of_nvlink_nominal": med / 900.0,
                            "seconds_per_step_max_rank": ar_time / max(1, len(tls))}
    return out


def cpu_baseline(model: dict, budget_layers: int | None = None) -> dict:
    """The oracle's CPU step (numpy, all host cores) on a bounded sample:
    one sample through `budget_layers` layers, fwd + bwd + SGD."""
    from oracle.executor_ref import CpuTrainer
    sub = dict(model)
    if budget_layers:
        sub["layers"] = budget_layers
    tr = CpuTrainer(sub)
    tr.step(0, 1)  # warm (BLAS threads, page-in)
    t0 = time.perf_counter()
    tr.step(1, 1)
    dt = time.perf_counter() - t0
    frac = sub["layers"] / model["layers"]
    return {"value": frac / dt, "unit": "samples/s", "cores": os.cpu_count(), "kind": "port",
            "sample": f"1 sample x {sub['layers']}/{model['layers']} layers fwd+bwd+SGD, fp32 numpy "
                      f"(oracle/executor_ref.py CpuTrainer), {dt:.2f}s"}


def run_reference(args, rank, world):
    """--impl reference: the CPU implementation of the step on this host."""
    if rank != 0:
        return
    model = MODELS[args.model]
    # VGG's loss needs the classifier: always the whole 19-layer net on one sample
    layers = model["layers"] if model["kind"] == "vgg" else min(model["layers"], args.ref_layers)
    from oracle.executor_ref import CpuTrainer
    sub = dict(model, layers=layers)
    tr = CpuTrainer(sub)
    for w in range(args.warmup):
        tr.step(w, 1)
    t0 = time.perf_counter()
    for k in range(args.steps):
        tr.step(args.warmup + k, 1)
    dt = time.perf_counter() - t0
    frac = layers / model["layers"]
    value = args.steps * frac / dt
    unit = "samples/s"
    line = {"metric": METRIC, "value": value, "unit": unit, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True,
            "scaling": "strong" if DEFAULTS[args.model]["straight"] or model["kind"] == "vgg" or
                                   "global_batch" in DEFAULTS[args.model] else "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic", "impl": "reference",
            "config": {"workload": args.model, **model},
            "cpu_baseline": {"value": value, "unit": unit, "cores": os.cpu_count(), "kind": "port",
                             "sample": f"each step: 1 sample x {layers}/{model['layers']} layers fwd+bwd+SGD, "
                                       "fp32 numpy oracle (the reference has no numerical executor)"},
            "e2e": {"value": value, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="dapple", choices=["dapple", "reference"])
    ap.add_argument("--model", default="bert48", choices=sorted(MODELS))
    ap.add_argument("--micro-batches", type=int, default=None, help="default per workload (DEFAULTS)")
    ap.add_argument("--slice", type=int, default=None, help="samples per replica slice of a micro-batch")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--ref-layers", type=int, default=8)
    ap.add_argument("--seed", type=int, default=1234)
    ap.add_argument("--plan", default="auto", choices=["auto", "forced", "planner"],
                    help="forced: [0,L)x1 / 2 stages x N/2 / straight; planner: the host planner's plan for the B200 "
                         "profile (profiled at its own replica slice sizes until the plan is a fixed point); "
                         "auto: planner for BERT-48 at N >= 2 (C2), forced otherwise")
    ap.add_argument("--mem-gb", type=float, default=None,
                    help="per_gpu_memory_gb given to the planner (default: 12 for BERT-48 -- pure DP needs 8 x P = "
                         "19.3 GB, so the planner must pipeline, as C2 does; 180 otherwise)")
    ap.add_argument("--global-batch", type=int, default=0, help="default: the workload's (BERT-48: 64 at every N)")
    ap.add_argument("--no-profile", action="store_true", help="skip the pre-run B200 layer profile")
    ap.add_argument("--schedule", default="dapple", choices=["dapple", "gpipe"])
    ap.add_argument("--recompute", action="store_true")
    ap.add_argument("--timeline-out", default=None,
                    help="write the last timed step's measured timeline (CSV + SVG, reference writers) here")
    args = ap.parse_args()
    dflt = DEFAULTS[args.model]
    args.micro_batches = args.micro_batches or dflt["micro_batches"]
    args.slice = args.slice or dflt["slice"]
    rank, world = dist_setup()
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE {world}")

    import torch
    torch.cuda.set_device(rank)
    from paper_2007_01045_b200 import _lib
    from paper_2007_01045_b200.runtime import Executor, merge_timelines

    from paper_2007_01045_b200 import pipeplan
    model = MODELS[args.model]
    M = args.micro_batches
    straight = dflt["straight"]
    strong = straight or model["kind"] == "vgg" or "global_batch" in dflt  # fixed global batch at every N
    gbs = args.global_batch or dflt.get("global_batch") or M * args.slice
    if args.plan == "auto":
        args.plan = "planner" if args.model == "bert48" and world >= 2 else "forced"
    if args.mem_gb is None:
        args.mem_gb = 12.0 if args.model == "bert48" else 180.0
    # NVLink calibration (peer-copy sweep on rank 0) feeds the cluster's intra_bw / intra_latency
    link = calibrate_link() if rank == 0 and world >= 2 else None
    link = broadcast(link, world)
    cluster = b200_cluster(world, args.mem_gb, link)
    # pre-run B200 layer profile at the micro-batch size: the planner's input
    # and the source of the predicted L (a real prediction, made before the run)
    mb = gbs // M
    profiles = {}  # samples -> B200 layer profile at that size
    planner_info = None
    if not args.no_profile or args.plan == "planner":
        profiles[mb] = profile_model(model, mb) if rank == 0 else None
    if args.plan == "planner":
        plan = None
        if rank == 0:
            plan, planner_info = plan_fixed_point(model, profiles, mb, cluster, M)
        plan = broadcast(plan, world)
    else:
        plan = make_plan(world, model["layers"], straight, model["kind"], sum(model.get("convs", [16])))
    if profiles and rank == 0:
        for st in plan["stages"]:
            size = -(-mb // len(st["gpus"]))
            if size not in profiles:
                profiles[size] = profile_model(model, size)
    profiles = broadcast(profiles, world)
    profile = slice_profile(profiles, plan, mb) if profiles else None
    S = len(plan["stages"])
    r0 = len(plan["stages"][0]["gpus"])
    lib = _lib.lib()

    ex = Executor(model, plan, M, gbs, lr=1e-4, seed=args.seed, rank=rank, world=world, device=rank,
                  schedule=args.schedule, recompute=args.recompute)
    clocks = ClockSampler() if rank == 0 else None
    if clocks:
        clocks.start()
    for _ in range(args.warmup):
        ex.step()
    torch.cuda.synchronize()

    # ------------------------------------------------------------ timed (device)
    barrier(world)
    if clocks:
        clocks.mark("t_start")
    launches0 = lib.dpl_k_launch_count()
    t_wall0 = time.perf_counter()
    tls = []
    for _ in range(args.steps):
        ex.step()
        tls.append(ex.timeline())
    torch.cuda.synchronize()
    barrier(world)
    t_wall = time.perf_counter() - t_wall0
    launches = lib.dpl_k_launch_count() - launches0
    if clocks:
        clocks.mark("t_stop")
    clk = clocks.stop() if clocks else None

    all_tls = gather(tls, world)  # [rank][step]
    lat, bub, spans = [], [], []
    for k in range(args.steps):
        merged = merge_timelines([all_tls[r][k] for r in range(world)], M, S)
        lat.append(merged["latency"])
        bub.append(merged["bubble"])
        spans.append((merged["start"], merged["end"]))
    total_launches = sum(gather(launches, world))
    # device-timed: on each rank's own GPU timer, start of the first timed
    # step to the end of the last one; the job time is the max over ranks
    own = [all_tls[r][-1]["t0_ns"] * 1e-9 + all_tls[r][-1]["step_s"] - all_tls[r][0]["t0_ns"] * 1e-9
           for r in range(world)]
    device_s = max(own)
    value = args.steps * gbs / device_s

    # ------------------------------------------------------------ GEMM roofline (one profiled step)
    ex.gemm_profile(True)
    ex.step()
    prof = ex.gemm_profile_report()
    step_tl = ex.timeline()
    ex.gemm_profile(False)
    profs = gather({"prof": prof, "step_s": step_tl["step_s"]}, world)

    # ------------------------------------------------------------ e2e (public API, host buffers)
    e2e = None
    if not args.no_e2e:
        inp, tgt = host_batches(model, plan, rank, M, gbs // M, args.seed)
        # three pinned buffer pairs in rotation, as a data loader hands them in:
        # the captured step's copy nodes are re-pointed, never re-captured
        bufs = [(inp, tgt)] + [(None if inp is None else inp.clone().pin_memory(),
                                None if tgt is None else tgt.clone().pin_memory()) for _ in range(2)]
        for k in range(2):  # warm the H2D path: one captured graph per flag bank (banks alternate by step)
            ex.step(*bufs[k])
        graphs_before = ex.graphs()
        barrier(world)
        t0 = time.perf_counter()
        for k in range(args.steps):
            ex.step(*bufs[k % 3])  # H2D of the step's inputs/targets, D2H of the loss
        torch.cuda.synchronize()
        barrier(world)
        t_e2e = time.perf_counter() - t0
        h2d = (inp.numel() * inp.element_size() if inp is not None else 0) + \
            (tgt.numel() * tgt.element_size() if tgt is not None else 0)
        d2h = 4 if rank in plan["stages"][-1]["gpus"] else 0
        sums = gather((h2d, d2h, t_e2e), world)
        e2e = {"value": args.steps * gbs / max(s[2] for s in sums), "unit": "samples/s",
               "h2d_bytes_per_step": sum(s[0] for s in sums), "d2h_bytes_per_step": sum(s[1] for s in sums),
               "timing": "wall clock between barriers, 3 pinned host buffer pairs in rotation",
               "captures_during_timed_steps": ex.graphs() - graphs_before}

    info = ex.info
    ex.close()
    if rank != 0:
        return

    # ------------------------------------------------------------ report
    peaks, peaks_src = load_peaks()
    # the kernel timer's per-launch events (the innermost pair around each
    # GEMM launch on the compute stream); the per-shape table comes from the
    # GEMM profile's outer events
    # GEMM time = the union of the GEMM launches' intervals on each rank's
    # step timeline: the weight-gradient GEMMs run on a side stream beside
    # the dgrad chain, so launches overlap and the plain sum of their
    # durations counts the shared time twice (reported too, as
    # per_launch_sum_tflops); the bf16 epilogue pass of split-K GEMMs counts
    # as GEMM time
    g_flops, g_secs, g_sum = 0.0, 0.0, 0.0
    for pr in profs:
        for k in pr["prof"].get("kernels", []):
            if k["kernel"] == "gemm_bf16_tcgen05":
                g_flops += k.get("flops", 0.0) or k.get("tflops", 0.0) * 1e12 * k["seconds"]
                g_secs += k.get("busy_seconds", k["seconds"])
                g_sum += k["seconds"]
            elif k["kernel"] == "gemm_split_epilogue":
                g_secs += k.get("busy_seconds", k["seconds"])
                g_sum += k["seconds"]
    if g_secs == 0.0:
        g_flops = sum(p["prof"]["flops"] for p in profs)
        g_secs = sum(p["prof"]["seconds"] for p in profs)
    achieved = g_flops / g_secs / 1e12 if g_secs > 0 else 0.0
    peak = peaks.get("bf16_tflops_sustained", PEAKS_FALLBACK["bf16_tflops_sustained"])
    gemm_share = g_secs / sum(p["step_s"] for p in profs)
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "gemm_traffic.json")) as f:
            traffic = json.load(f).get("bytes_per_launch")
    except Exception:
        pass
    calib = calibrated_profile(model, plan, [all_tls[r][-1] for r in range(world)], profile)
    pred_cal = predicted_latency(plan, calib, cluster, M, world, args.schedule)
    pred = None
    if profile is not None:
        prof_run = profile
        if args.recompute:
            prof_run = {**profile, "layers": [{**l, "bwd_time_us": l["bwd_time_us"] + l["fwd_time_us"]}
                                              for l in profile["layers"]]}  # apply_recompute, simulator.cpp:216-221
        pred = predicted_latency(plan, prof_run, cluster, M, world, args.schedule)
    phi_tl = info["phi_expanded"] if args.schedule == "dapple" else [M] * (2 * S - 1)
    exported = pipeplan.timeline_export(merge_timelines([all_tls[r][-1] for r in range(world)], M, S), M,
                                        2 * S - 1, phi_tl, plan, calib, cluster)
    if args.timeline_out:
        os.makedirs(args.timeline_out, exist_ok=True)
        for size, pr in profiles.items():  # the B200 profiles, in the reference's profile format
            with open(os.path.join(args.timeline_out, f"profile_{args.model}_mb{size}.json"), "w") as f:
                f.write(pipeplan.call("load_profile", profile=json.dumps(pr))["json"])
        tag = f"{args.model}_n{world}_{args.schedule}{'_rc' if args.recompute else ''}"
        with open(os.path.join(args.timeline_out, f"timeline_{tag}.csv"), "w") as f:
            f.write(exported["csv"])
        with open(os.path.join(args.timeline_out, f"timeline_{tag}.svg"), "w") as f:
            f.write(exported["svg"])
    measured_ms = statistics.mean(lat) * 1e3
    fps = flops_per_sample(model)
    line = {
        "metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": measured_ms, "higher_is_better": True,
        "scaling": "strong" if strong else "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic (seeded splitmix64 inputs/targets, random-init "
                                                      "weights)",
        "config": {"workload": args.model, **model, "global_batch": gbs, "micro_batches": M,
                   "plan_source": "host planner (pipeplan.plan on the B200 profile, per_gpu_memory_gb="
                                  f"{args.mem_gb:g})" if args.plan == "planner" else "forced",
                   "plan": [[s["layers"], s["gpus"]] for s in plan["stages"]],
                   "phi": info["phi_expanded"], "parallelism": f"{S} stages x {r0} replicas",
                   "l2": "working set (GBs of activations) far larger than the 126 MB L2"},
        "bubble": statistics.mean(bub),
        "device_s": device_s,
        "schedule": {"kind": args.schedule, "recompute": args.recompute, "stash_slots": info["stash_slots"],
                     "peak_activations_measured": exported["peak_activations"],
                     "device_bytes": info.get("device_bytes")},
        "comm": comm_stats([all_tls[r][-1] for r in range(world)], link),
        "link_calibration": link,
        "latency": {"measured_ms": measured_ms,
                    "planner": None if planner_info is None else {
                        **planner_info, "measured_over_planner_sim": measured_ms / planner_info["sim_latency_ms"],
                        "measured_over_planner_est": measured_ms / planner_info["est_latency_ms"]},
                    "predicted": None if pred is None else {
                        **pred, "measured_over_sim": measured_ms / pred["sim_ms"],
                        "profile": "B200 layer profiles taken before the run (Executor.layer_profile) at "
                                   f"the replica slice sizes {sorted(profiles)}, planner cost model"},
                    "calibrated": {**pred_cal, "measured_over_sim": measured_ms / pred_cal["sim_ms"],
                                   "profile": "per-layer F/B from this run's measured blocks"}},
        "tflops_per_gpu": fps * value / world / 1e12,
        "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "kernel": "gemm_bf16_tcgen05 (all launches of one step, CUDA events around each launch; "
                               "time = union of the launch intervals)",
                     "per_launch_sum_tflops": g_flops / g_sum / 1e12 if g_sum > 0 else 0.0,
                     "peak_source": f"bf16_tflops_sustained of {peaks_src}", "gemm_share_of_step": gemm_share,
                     "shapes": prof["shapes"][:16]},
        "kernels": sorted(prof.get("kernels", []), key=lambda k: -k["seconds"]),
        "clocks": clk,
        "gpu_launches": total_launches,
        "wall_s": t_wall,
        "e2e": e2e,
    }
    if world == 1 and not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline(model, budget_layers=min(model["layers"], 48))
        if profile is not None:
            # the reference planner + simulator beside the new host planner on
            # the C2 planning problem built from this run's B200 profile
            try:
                c2 = b200_cluster(8, 12.0)
                c2_plan = pipeplan.plan(profile, c2, M)["plan"]
                line["cpu_baseline"]["planner"] = planner_cpu_times(profile, c2, M, c2_plan)
            except Exception as e:  # noqa: BLE001 -- a missing checker must not cost the line
                line["cpu_baseline"]["planner"] = {"error": str(e)[:200]}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
