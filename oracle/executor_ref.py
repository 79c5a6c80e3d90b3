"""CPU numerical oracle for the DAPPLE training step (TEST INFRASTRUCTURE ONLY).

The reference has no numerical executor (loss/gradient
parity is *unpinned* by any reference test).  This module restates the
step's semantics from the paper's runtime section:

* forward graphs per stage in order, backward graphs in reverse order
  (PAPER.md:1192-1201);
* a micro-batch is split into even row slices over a stage's replicas, with
  split/concat at stage boundaries;
* every device accumulates gradients over all its micro-batches, then an
  AllReduce over the replicas, then Apply;
* so the step equals full-batch training at fixed GBS.

It is pinned internally: ``scheduled_step`` (which walks the exact per-stage
1F1B chain of the plan, slices micro-batches per replica and accumulates
per replica) must equal ``full_batch_step`` (one sequential fp64 pass) to
rounding -- tests/test_oracle_executor.py.  The GPU executor is then checked
against ``full_batch_step`` in fp32 within the bf16 tolerance stated in the
tests.

Synthetic data and weights come from ``hash_uniform`` -- the same splitmix64
keyed generator the device uses (csrc/kernels/elementwise.cu), so the oracle
and the GPU see identical inputs without shipping tensors.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

_K_TENSOR = np.uint64(0xD1B54A32D192ED03)
_K_INDEX = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D649BB133111EB)


def hash_uniform(seed: int, tensor: int, idx) -> np.ndarray:
    """U(-1, 1) float32 keyed by (seed, tensor id, element index)."""
    idx = np.asarray(idx, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(seed) + np.uint64(tensor) * _K_TENSOR + idx * _K_INDEX
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        z = z ^ (z >> np.uint64(31))
    u = (z >> np.uint64(40)).astype(np.float32) * np.float32(1.0 / 16777216.0)
    return u * np.float32(2.0) - np.float32(1.0)
