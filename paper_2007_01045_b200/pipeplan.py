"""Python mirror of the reference's pipeplan API (proj/include/pipeplan/*.hpp),
backed by the C++ host library in libdapple.so (dpl_host_call).

Function names, argument meaning and error behaviour follow the reference:
errors raise the Python counterpart of the reference's exception class
(ValueError for std::invalid_argument, IndexError for std::out_of_range,
RuntimeError for std::runtime_error / std::logic_error), carrying the
reference's message.  Units in the returned dicts are seconds and bytes, as
in the reference's in-memory types; the *_us fields of plans are the file
format (io.cpp:23-38).
"""
from __future__ import annotations

import json
from typing import Any

from ._lib import lib  # noqa: F401  (re-exported for tests)

_ERRORS = {"invalid_argument": ValueError, "out_of_range": IndexError, "runtime_error": RuntimeError,
           "logic_error": RuntimeError}


class PipeplanError(RuntimeError):
    pass


def call(op: str, **kwargs: Any) -> dict:
    req = {"op": op}
    req.update(kwargs)
    reply = json.loads(lib().dpl_host_call(json.dumps(req).encode()))
    if "error" in reply:
        err = reply["error"]
        raise _ERRORS.get(err["type"], PipeplanError)(err["what"])
    return reply


def plan(profile, cluster, micro_batches, phi_strategy="preset_a", top_k=8, optimizer_multiplier=8.0, report=False):
    """planner.hpp:71-73 -> {"plan": {...}, "report": {...}?}"""
    return call("plan", profile=profile, cluster=cluster, M=micro_batches, phi_strategy=phi_strategy, top_k=top_k,
                optimizer_multiplier=optimizer_multiplier, report=report)


def brute_force_plan(profile, cluster, micro_batches, phi_strategy="preset_a"):
    return call("brute_force_plan", profile=profile, cluster=cluster, M=micro_batches, phi_strategy=phi_strategy)


def simulate_plan(plan_json, profile, cluster, micro_batches, schedule="dapple", recompute=False):
    """planner.hpp:87-90 -> {"latency", "seq", "timeline", "peaks", "csv"}"""
    return call("simulate_plan", plan=plan_json, profile=profile, cluster=cluster, M=micro_batches,
                schedule=schedule, recompute=recompute)


def build_stage_sequence(plan_json, profile, cluster):
    return call("build_stage_sequence", plan=plan_json, profile=profile, cluster=cluster)["seq"]


def estimate_latency(seq, micro_batches):
    return call("estimate", seq=seq, M=micro_batches)


def dapple_schedule(seq, micro_batches, phi):
    return call("schedule", seq=seq, M=micro_batches, phi=phi)


def gpipe_schedule(seq, micro_batches):
    return call("schedule", seq=seq, M=micro_batches, schedule="gpipe")


def optimize_phi(seq, micro_batches, strategy, max_injection):
    return call("optimize_phi", seq=seq, M=micro_batches, phi_strategy=strategy, D=max_injection)


def expand_plan_phi(phi):
    return call("expand_plan_phi", phi=phi)["phi"]


def stage_chain(micro_batches, phi, schedule="dapple"):
    return [("F" if k == 0 else "B", i) for k, i in call("stage_chain", M=micro_batches, phi=phi,
                                                          schedule=schedule)["chain"]]


def allreduce_time(size, devices, cluster):
    return call("allreduce_time", size=size, devices=devices, cluster=cluster)["t"]


def splitconcat_time(size, src, dst, cluster):
    return call("splitconcat_time", size=size, src=src, dst=dst, cluster=cluster)["t"]


def enumerate_placements(cluster, count, free=None):
    kw = {} if free is None else {"free": free}
    return call("enumerate_placements", cluster=cluster, count=count, **kw)["placements"]


def timeline_export(timeline, micro_batches, stage_count, phi, plan_json=None, profile=None, cluster=None):
    """A measured timeline (runtime.merge_timelines) through the reference's
    writers: {"csv": write_timeline_csv (io.cpp), "peak_activations"
    (simulator.cpp), and with plan/profile/cluster also "svg"
    (write_timeline_svg) and "latency" (batch_latency)}.  Times are shifted
    so the first forward starts at 0, as in a simulated timeline."""
    import math
    blocks = [b for b in timeline["blocks"] if not math.isnan(b[3])]
    t0 = min(b[3] for b in blocks) if blocks else 0.0
    req = {"timeline": {"M": micro_batches, "S": stage_count, "phi": list(phi),
                        "blocks": [[x, i, k, s - t0, e - t0] for x, i, k, s, e in blocks]}}
    if plan_json is not None:
        req.update(plan=plan_json, profile=profile, cluster=cluster)
    return call("timeline_export", **req)
