"""Bit-exact planner / estimator / simulator parity with the reference.

* golden fixtures produced by the compiled reference (tests/golden/
  make_golden.py): every reply of the product library must equal the
  reference's reply exactly (parsed doubles, plans, timelines, CSV text,
  error class and message);
* a live differential against oracle/_ref/ref_cli on fresh random instances
  when the reference build is present;
* explicit restatements of the reference's own unit-test assertions.
"""
import json
import os
import random

import pytest

from paper_2007_01045_b200 import pipeplan

HERE = os.path.dirname(os.path.abspath(__file__))


def _golden():
    with open(os.path.join(HERE, "golden", "planner_golden.json")) as f:
        return json.load(f)


GOLDEN = _golden()


def _mine(req):
    r = {k: v for k, v in req.items() if k != "tag"}
    return json.loads(pipeplan.lib().dpl_host_call(json.dumps(r).encode()))


def _norm(reply):
    """Serialized profile/cluster documents are compared as parsed JSON
    (whitespace of nlohmann's pretty printer is not part of the contract)."""
    if isinstance(reply, dict) and isinstance(reply.get("json"), str):
        reply = dict(reply, json=json.loads(reply["json"]))
    return reply


@pytest.mark.parametrize("case", range(len(GOLDEN)))
def test_golden_case(case):
    g = GOLDEN[case]
    assert _norm(_mine(g["request"])) == _norm(g["response"]), g["request"].get("tag", g["request"]["op"])


def test_live_differential_random():
    oracle = pytest.importorskip("oracle.refproc")
    if not oracle.available():
        pytest.skip("reference build absent (oracle/_ref)")
    ref = oracle.shared()
    rng = random.Random(4242)
    for _ in range(40):
        n = rng.randint(1, 11)
        prof = {"profile_batch_size": 1, "layers": [
            {"fwd_time_us": rng.uniform(200, 4000), "bwd_time_us": 2 * rng.uniform(200, 4000),
             "activation_bytes": rng.randint(0, 8 << 20), "param_bytes": rng.randint(0, 4 << 20)} for _ in range(n)]}
        seps = rng.choice([[1], [2], [3], [4], [1, 1], [2, 2], [1, 3], [2, 1], [1, 1, 1], [4, 4], [8]])
        cl = {"seps": seps, "intra_bw_gbps": 80, "inter_bw_gbps": 8, "intra_latency_us": 1, "inter_latency_us": 10,
              "per_gpu_memory_gb": 16}
        req = {"op": "plan", "profile": prof, "cluster": cl, "M": 4 + rng.randint(0, 4),
               "phi_strategy": rng.choice(["preset_a", "preset_b", "search"]), "report": True}
        assert _mine(req) == ref.call(req)
        if sum(seps) <= 4 and n <= 8:
            req["op"] = "brute_force_plan"
            assert _mine(req) == ref.call(req)


def _seq(f, b, ar=None):
    return [{"kind": "compute", "fwd": x, "bwd": y, "allreduce": (ar[i] if ar else 0.0)}
            for i, (x, y) in enumerate(zip(f, b))]


def _block(tl, x, i, kind):
    S, M = tl["S"], tl["M"]
    idx = x * M + i if kind == 0 else S * M + x * M + i
    return tl["blocks"][idx]


def test_reference_unit_assertions():
    # simulator_test.cpp:29-52 frozen 2x2 trace
    r = pipeplan.dapple_schedule(_seq([1, 1], [1, 1]), 2, [2, 1])
    tl = r["timeline"]
    assert _block(tl, 1, 1, 0)[3:] == [3.0, 4.0] and _block(tl, 0, 1, 1)[3:] == [5.0, 6.0]
    assert r["latency"] == 6.0 and r["peaks"] == [2, 1]
    # simulator_test.cpp:54-59 / estimator_test.cpp:109-116 even 4-stage L = 30
    assert pipeplan.dapple_schedule(_seq([1] * 4, [2] * 4), 7, [4, 3, 2, 1])["latency"] == pytest.approx(30.0)
    est = pipeplan.estimate_latency(_seq([1] * 4, [2] * 4), 7)
    assert (est["warmup"], est["steady"], est["ending"], est["pivot"]) == (4.0, 18.0, 8.0, 3)
    # estimator_test.cpp:117-126 unbalanced middle pivot, L = 39
    est = pipeplan.estimate_latency(_seq([1, 3, 1], [2, 6, 2]), 4)
    assert est["pivot"] == 1 and est["total"] == pytest.approx(39.0)
    # simulator_test.cpp:217-242 presets
    s5 = _seq([1] * 5, [2] * 5)
    assert pipeplan.optimize_phi(s5, 16, "preset_a", 16)["phi"] == [5, 4, 3, 2, 1]
    assert pipeplan.optimize_phi(s5, 16, "preset_b", 16)["phi"] == [9, 7, 5, 3, 1]
    assert pipeplan.optimize_phi(s5, 16, "preset_a", 3)["phi"] == [3, 3, 3, 2, 1]
    assert pipeplan.optimize_phi(s5, 2, "preset_b", 16)["phi"] == [2, 2, 2, 2, 1]
    # simulator_test.cpp:258-262
    assert pipeplan.expand_plan_phi([3, 2, 1]) == [3, 2, 2, 1, 1]
    # costmodel_test.cpp:37-41, 65-80
    c2 = {"seps": [2], "intra_bw_gbps": 100, "inter_bw_gbps": 10, "intra_latency_us": 0, "inter_latency_us": 0,
          "per_gpu_memory_gb": 16}
    assert pipeplan.allreduce_time(10**9, [0, 1], c2) == pytest.approx(0.01)
    c88 = dict(c2, seps=[8, 8], inter_latency_us=2)
    assert pipeplan.splitconcat_time(10**9, [0], [8, 9], c88) == pytest.approx(0.05 + 2e-6)
    # planner_test.cpp:84-107 placements
    c16 = dict(c2, seps=[8, 8], intra_latency_us=1, inter_latency_us=10)
    assert pipeplan.enumerate_placements(c16, 8)[0] == list(range(8))
    assert [4, 5, 6, 7] in pipeplan.enumerate_placements(c16, 4, free=[4, 8])
    assert [0, 8] in pipeplan.enumerate_placements(c16, 2)
    # errors keep the reference's classes and messages
    with pytest.raises(ValueError, match="phi must be non-increasing"):
        pipeplan.dapple_schedule(_seq([1] * 3, [1] * 3), 4, [2, 3, 1])
    with pytest.raises(RuntimeError, match="enumerate_placements: insufficient free GPUs"):
        pipeplan.enumerate_placements(c16, 17)


def test_stage_chain_matches_survey_order():
    # phi_exp=[3,2,1], M=8, stage 0
    chain = pipeplan.stage_chain(8, 3)
    assert " ".join(f"{k}{i}" for k, i in chain) == "F0 F1 F2 B0 F3 B1 F4 B2 F5 B3 F6 B4 F7 B5 B6 B7"
    assert [k for k, _ in pipeplan.stage_chain(4, 1, "gpipe")] == ["F"] * 4 + ["B"] * 4


@pytest.mark.parametrize("b_mb,ra,rb", [(6, 3, 1), (6, 1, 3), (12, 4, 3), (8, 2, 4), (8, 4, 4),
                                        (8, 1, 7), (8, 7, 1), (7, 2, 3), (5, 5, 4), (9, 4, 6)])
def test_splitconcat_routes_partition_the_rows(b_mb, ra, rb):
    plan = {"stages": [{"layers": [0, 1], "gpus": list(range(ra))},
                       {"layers": [1, 2], "gpus": list(range(ra, ra + rb))}]}
    routes = pipeplan.call("splitconcat_routes", plan=plan, boundary=0, micro_batch=b_mb, rows_per_sample=512)["routes"]
    assert len(routes) <= ra + rb - 1
    # replica j owns samples [b*j/r, b*(j+1)/r) (uneven when r does not divide b)
    covered = sorted((b_mb * s // ra * 512 + so, r) for s, d, so, do, r in routes)
    pos = 0
    for start, rows in covered:  # source rows are covered exactly once, in order
        assert start == pos
        pos += rows
    assert pos == b_mb * 512
    dst = sorted((b_mb * (d - ra) // rb * 512 + do, r) for s, d, so, do, r in routes)
    pos = 0
    for start, rows in dst:
        assert start == pos
        pos += rows
    assert pos == b_mb * 512


def test_splitconcat_routes_reject_more_replicas_than_samples():
    plan = {"stages": [{"layers": [0, 1], "gpus": [0, 1, 2]}, {"layers": [1, 2], "gpus": [3]}]}
    with pytest.raises(ValueError):
        pipeplan.call("splitconcat_routes", plan=plan, boundary=0, micro_batch=2, rows_per_sample=1)


def test_timeline_export_reproduces_reference_writers():
    """The exporter used for MEASURED timelines (bench --timeline-out) goes
    through the same write_timeline_csv / peak_activations / batch_latency as
    the reference: fed each golden simulate_plan timeline it must return the
    reference's own CSV, peaks and latency byte for byte."""
    cases = [g for g in GOLDEN if g["request"]["op"] == "simulate_plan"]
    assert cases
    for g in cases:
        req, want = g["request"], g["response"]
        tl = want["timeline"]
        got = pipeplan.call("timeline_export", timeline=tl, plan=req["plan"], profile=req["profile"],
                            cluster=req["cluster"])
        assert got["csv"] == want["csv"]
        assert got["peak_activations"] == want["peaks"]
        if not req.get("recompute"):
            assert got["latency"] == want["latency"]
        assert got["svg"].startswith("<svg")


def test_parallel_search_is_bit_identical_to_sequential():
    """plan() expands BFS batches on worker threads (DPL_PLANNER_THREADS) and
    replays leaderboard offers / memo decisions in FIFO order: the plan and
    the whole top-k report must equal the single-threaded search's."""
    import subprocess
    import sys
    code = """
import json, random, sys
sys.path.insert(0, %r)
from paper_2007_01045_b200 import pipeplan
r = random.Random(7)
prof = {"profile_batch_size": 8, "layers": [{"fwd_time_us": r.uniform(100, 1000), "bwd_time_us": r.uniform(200, 2000),
        "activation_bytes": r.randint(1 << 20, 1 << 26), "param_bytes": r.randint(1 << 20, 1 << 27)} for _ in range(20)]}
cl = {"seps": [4, 4], "intra_bw_gbps": 300.0, "inter_bw_gbps": 25.0, "intra_latency_us": 5.0,
      "inter_latency_us": 10.0, "per_gpu_memory_gb": 40.0}
print(json.dumps(pipeplan.plan(prof, cl, 8, report=True), sort_keys=True))
""" % os.path.dirname(HERE)
    outs = []
    for threads in ("1", "4"):
        env = dict(os.environ, DPL_PLANNER_THREADS=threads)
        outs.append(subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env,
                                   check=True).stdout)
    assert outs[0] == outs[1]
    assert json.loads(outs[0])["report"]["states_evaluated"] > 10000
