"""Per-GPU executor driver: the B200 counterpart of simulate_plan
(reference planner.hpp:87-90).  One process per GPU; torch.distributed is
used only for plumbing (exchanging CUDA-IPC handles and NCCL ids).  The step
itself -- the plan's early-backward 1F1B chain, Split-Concat peer copies,
per-layer NCCL AllReduce and SGD apply -- runs in libdapple.so (C++/CUDA).
"""
from __future__ import annotations

import ctypes
import json
import math
import os
from typing import Optional

from ._lib import check, lib

BLOB_BYTES = 256  # PeerBlob (executor.cu): IPC handles + pid / device / pointers


class Executor:
    def __init__(self, model: dict, plan, micro_batches: int, gbs: int, *, lr: float = 1e-3, seed: int = 1234,
                 rank: int = 0, world: int = 1, device: Optional[int] = None, apply: bool = True,
                 timeline: bool = True, schedule: str = "dapple", recompute: bool = False,
                 allreduce: Optional[str] = None, connect: bool = True, probe: bool = False,
                 wgrad_stream: Optional[bool] = None):
        self.plan = json.loads(plan) if isinstance(plan, str) else plan
        self.model, self.M, self.gbs = model, micro_batches, gbs
        self.rank, self.world = rank, world
        self.device = rank if device is None else device
        self.allreduce = allreduce or os.environ.get("DPL_ALLREDUCE", "peer")
        cfg = {"model": model, "plan": self.plan, "M": micro_batches, "gbs": gbs, "lr": lr, "seed": seed,
               "rank": rank, "world": world, "apply": apply, "timeline": timeline,
               "schedule": schedule, "recompute": recompute, "allreduce": self.allreduce, "probe": probe,
               "graph": os.environ.get("DPL_GRAPH", "1") != "0"}
        if wgrad_stream is not None:
            cfg["wgrad_stream"] = wgrad_stream
        h = ctypes.c_void_p()
        check(lib().dpl_exec_create(json.dumps(cfg).encode(), self.device, ctypes.byref(h)))
        self._h = h
        self.info = self._info()
        self.clock_offsets_ns = [0] * world
        if world > 1 and connect:
            self._connect()

    # ----------------------------------------------------------- plumbing
    def _info(self) -> dict:
        buf = ctypes.create_string_buffer(1 << 16)
        check(lib().dpl_exec_info(self._h, buf, len(buf)))
        return json.loads(buf.value.decode())

    def export(self) -> bytes:
        blob = ctypes.create_string_buffer(BLOB_BYTES)
        n = ctypes.c_size_t()
        check(lib().dpl_exec_export(self._h, blob, BLOB_BYTES, ctypes.byref(n)))
        return bytes(blob.raw[:BLOB_BYTES])

    def connect_blobs(self, blobs: list):
        check(lib().dpl_exec_connect(self._h, b"".join(blobs), BLOB_BYTES, self.world))

    def _connect(self):
        import torch.distributed as dist
        blobs = [None] * self.world
        dist.all_gather_object(blobs, self.export())
        self.connect_blobs(blobs)
        # NCCL mode: one communicator per stage replica group; its first GPU makes the id
        stage = self.plan["stages"][self.info["stage"]]
        leader = sorted(stage["gpus"])[0]
        nccl = self.allreduce == "nccl" and len(stage["gpus"]) > 1
        my_id = None
        if self.rank == leader and nccl:
            idbuf = ctypes.create_string_buffer(128)
            check(lib().dpl_exec_nccl_id(idbuf))
            my_id = bytes(idbuf.raw)
        ids = [None] * self.world
        dist.all_gather_object(ids, my_id)
        if nccl:
            check(lib().dpl_exec_nccl_init(self._h, ids[leader]))
        self.clock_offsets_ns = self._calibrate_clocks()

    def _calibrate_clocks(self):
        """%globaltimer differs between GPUs; rank 0 ping-pongs every peer over
        NVLink peer memory and the offsets are shared, so merged timelines are
        on rank 0's clock."""
        import threading
        import torch.distributed as dist
        offsets = [0] * self.world
        for phase in range(1, self.world):
            off = ctypes.c_longlong(0)
            if self.rank == phase:
                # responder first: it zeroes its words, then spins for pings
                dist.barrier()
                check(lib().dpl_exec_clock_calibrate(self._h, phase, ctypes.byref(off)))
            elif self.rank == 0:
                dist.barrier()
                check(lib().dpl_exec_clock_calibrate(self._h, phase, ctypes.byref(off)))
                offsets[phase] = off.value
            else:
                dist.barrier()
            dist.barrier()
        allv = [None] * self.world
        dist.all_gather_object(allv, offsets if self.rank == 0 else None)
        return allv[0]

    # ----------------------------------------------------------- step
    def step(self, host_input=None, host_target=None) -> float:
        """One synchronous DAPPLE step.  host_input / host_target: pinned host
        tensors holding this replica's slices of every micro-batch
        ([M][rows][H] bf16), or None to generate the seeded synthetic data on
        the device.  Returns the global-batch loss on last-stage ranks."""
        loss = ctypes.c_float(float("nan"))
        pin = self._host_arg(host_input, "input")
        pt = self._host_arg(host_target, "target")
        check(lib().dpl_exec_step(self._h, pin, pt, ctypes.byref(loss)))
        return loss.value

    def _host_arg(self, t, which: str):
        """Validates one step's host tensor (this rank's slices of every
        micro-batch) and returns its address.  Pinned memory is read in place
        by the captured step; pageable memory is staged by the library."""
        if t is None:
            return None
        want = self.info[f"{which}_bytes"]
        if want == 0:  # this rank's stage does not consume it (e.g. targets on stage 0)
            return None
        import numpy as np
        import torch
        if isinstance(t, np.ndarray):
            t = torch.from_numpy(t)
        if not isinstance(t, torch.Tensor):
            raise TypeError(f"{which}: expected a torch.Tensor or numpy array, got {type(t).__name__}")
        if t.device.type != "cpu":
            raise ValueError(f"{which}: host tensor expected, got device {t.device}")
        dtype = {"int32": torch.int32, "bfloat16": torch.bfloat16}[self.info[f"{which}_dtype"]]
        if t.dtype != dtype:
            raise TypeError(f"{which}: dtype {t.dtype}, expected {dtype}")
        if not t.is_contiguous():
            raise ValueError(f"{which}: tensor must be contiguous")
        if t.numel() * t.element_size() != want:
            raise ValueError(f"{which}: {t.numel() * t.element_size()} bytes, expected {want} "
                             f"([M={self.M}] x this replica's slice)")
        if dtype == torch.int32:
            hi = self.model.get("vocab") if (which == "input" or self.model.get("vocab")) else self.model.get("classes")
            lo_v, hi_v = int(t.min()), int(t.max())
            if lo_v < 0 or (hi and hi_v >= hi):
                raise ValueError(f"{which}: ids must lie in [0, {hi}), got [{lo_v}, {hi_v}]")
        return ctypes.c_void_p(t.data_ptr())

    def graphs(self) -> int:
        """Captured step graphs held (one per flag bank x host-data mode)."""
        return self._info()["graphs"]

    def step_launch(self, host_input=None, host_target=None):
        """Enqueues one step and returns at once (see LocalRanks)."""
        self._keep = (host_input, host_target)
        check(lib().dpl_exec_step_launch(self._h, self._host_arg(host_input, "input"),
                                         self._host_arg(host_target, "target")))

    def step_finish(self) -> float:
        loss = ctypes.c_float(float("nan"))
        check(lib().dpl_exec_step_finish(self._h, ctypes.byref(loss)))
        self._keep = None
        return loss.value

    def gemm_profile(self, enable: bool):
        check(lib().dpl_exec_gemm_profile(self._h, int(enable)))

    def layer_profile(self, reps: int = 5) -> dict:
        """This stage's layers timed on the GPU at this replica's micro-batch
        slice, as the reference's profile JSON (model.cpp:162-173)."""
        out = lib().dpl_exec_layer_profile(self._h, reps)
        if out is None:
            raise RuntimeError(lib().dpl_last_error().decode())
        return json.loads(out.decode())

    def gemm_profile_report(self) -> dict:
        return json.loads(lib().dpl_exec_gemm_profile_json(self._h).decode())

    def timeline(self) -> dict:
        tl = json.loads(lib().dpl_exec_timeline(self._h).decode())
        # express t0 on rank 0's GPU timer
        tl["t0_ns"] -= getattr(self, "clock_offsets_ns", [0] * self.world)[self.rank]
        return tl

    def read(self, layer: int, name: str, count: int, grad: bool = False):
        import numpy as np
        out = np.empty(count, dtype=np.float32)
        check(lib().dpl_exec_read_tensor(self._h, f"{layer}.{name}".encode(), int(grad),
                                         out.ctypes.data_as(ctypes.c_void_p), out.nbytes))
        return out

    def probe(self, layer: int, which: str, count: int):
        """Teacher-forcing probe (Executor(..., probe=True)): the last
        micro-batch's x / y / aux / dy / dx of `layer`, as float32."""
        import numpy as np
        import torch
        out = torch.empty(count, dtype=torch.bfloat16)
        check(lib().dpl_exec_read_probe(self._h, layer, which.encode(), ctypes.c_void_p(out.data_ptr()),
                                        count * 2))
        return out.float().numpy().astype(np.float64)

    def close(self):
        """Collective when world > 1: unmap peers, barrier, then free."""
        if getattr(self, "_h", None):
            if self.world > 1:
                import torch.distributed as dist
                check(lib().dpl_exec_disconnect(self._h))
                if dist.is_initialized():
                    dist.barrier()
            lib().dpl_exec_destroy(self._h)
            self._h = None

    def __del__(self):
        # never collective from a finaliser: just free local state
        if getattr(self, "_h", None):
            try:
                lib().dpl_exec_destroy(self._h)
            except Exception:
                pass
            self._h = None


class LocalRanks:
    """Every rank of a plan in this one process (several ranks may share one
    GPU, e.g. all on cuda:0): the ranks map each other's receive regions and
    gradients with plain pointers instead of CUDA IPC, their flag waits stay
    stream memory operations, and the replica AllReduce runs over the shared
    memory (collective.cu) -- the same step program as one process per GPU,
    so the Split-Concat hand-off, the cross-rank flag chain and the replica
    reduction are exercised on a single device.  A step launches every
    rank's captured step, then waits for all of them."""

    def __init__(self, model: dict, plan, micro_batches: int, gbs: int, *, devices=None, **kw):
        # Before CUDA initialises: kernels loaded eagerly (lazy loading
        # synchronises the context on a kernel's first launch, deadlocking
        # ranks that wait on each other) and one hardware work queue per
        # stream (ranks' blocked flag waits must not sit in front of another
        # rank's work).
        want = {"CUDA_MODULE_LOADING": "EAGER", "CUDA_DEVICE_MAX_CONNECTIONS": "32"}
        if any(os.environ.get(k) != v for k, v in want.items()):
            import torch
            if torch.cuda.is_initialized():
                raise RuntimeError("LocalRanks needs CUDA_MODULE_LOADING=EAGER and CUDA_DEVICE_MAX_CONNECTIONS=32 "
                                   "set before CUDA initialises")
            os.environ.update(want)
        plan = json.loads(plan) if isinstance(plan, str) else plan
        world = 1 + max(g for s in plan["stages"] for g in s["gpus"])
        devices = devices or [0] * world
        if kw.get("allreduce", "peer") != "peer":
            raise ValueError("LocalRanks reduce over shared memory (allreduce='peer')")
        # The weight-gradient side stream stays off here: with several ranks'
        # step graphs co-resident in one context, its extra branch can share a
        # hardware queue with another rank's blocked flag wait (observed as a
        # hang on one B200); one process per GPU has no such sharing.
        kw.setdefault("wgrad_stream", False)
        self.ranks = [Executor(model, plan, micro_batches, gbs, rank=r, world=world, device=devices[r],
                               allreduce="peer", connect=False, **kw) for r in range(world)]
        blobs = [ex.export() for ex in self.ranks]
        for ex in self.ranks:
            ex.connect_blobs(blobs)
        # every rank's step graphs exist before any rank runs
        for ex in self.ranks:
            check(lib().dpl_exec_prepare(ex._h))
        self.world = world

    def step(self, inputs=None, targets=None) -> list:
        """One step on every rank; returns the per-rank losses (NaN except on
        last-stage ranks)."""
        inputs = inputs or [None] * self.world
        targets = targets or [None] * self.world
        for ex, x, t in zip(self.ranks, inputs, targets):
            ex.step_launch(x, t)
        return [ex.step_finish() for ex in self.ranks]

    def timelines(self) -> list:
        return [ex.timeline() for ex in self.ranks]

    def close(self):
        for ex in self.ranks:  # unmap peers everywhere before anyone frees
            if getattr(ex, "_h", None):
                check(lib().dpl_exec_disconnect(ex._h))
        for ex in self.ranks:
            if getattr(ex, "_h", None):
                lib().dpl_exec_destroy(ex._h)
                ex._h = None


def merge_timelines(parts: list, micro_batches: int, stages: int) -> dict:
    """Combines per-rank measured timelines into one Timeline over the
    expanded 2S-1 stages (simulator.hpp:25-35 layout), aligned on the GPUs'
    global timer.  A replicated stage's block spans its replicas (min start,
    max end).  Returns {"blocks", "latency", "busy", "bubble"}."""
    t0 = min(p["t0_ns"] for p in parts) * 1e-9
    se = 2 * stages - 1
    span = {}
    for p in parts:
        off = p["t0_ns"] * 1e-9 - t0
        for x, i, kind, s, e in p["blocks"]:
            if s < 0 or e < 0:
                continue
            key = (x, i, kind)
            s, e = s + off, e + off
            if key in span:
                span[key] = (min(span[key][0], s), max(span[key][1], e))
            else:
                span[key] = (s, e)
    blocks = []
    for x in range(se):
        for kind in (0, 1):
            for i in range(micro_batches):
                s, e = span.get((x, i, kind), (math.nan, math.nan))
                blocks.append([x, i, kind, s, e])
    # measured L: first forward start -> end of the last rank's step (apply,
    # AllReduce and hand-offs drained), on the GPUs' global timer
    first = min(s for x, i, k, s, e in blocks if k == 0 and x % 2 == 0 and not math.isnan(s))
    end = max(p["t0_ns"] * 1e-9 - t0 + p["step_s"] for p in parts)
    latency = end - first
    busy = sum(sum(e - s for x, i, k, s, e in p["blocks"] if x % 2 == 0 and s >= 0) for p in parts)
    return {"blocks": blocks, "latency": latency, "start": first + t0, "end": end + t0, "busy": busy,
            "bubble": 1.0 - busy / (len(parts) * latency)}
