"""CPU checks of bench.py's workload helpers and the measured-timeline merge
(no GPU): plan shapes per workload, FLOP accounting against SURVEY.md
§8(d), slice profiles, and runtime.merge_timelines on synthetic blocks."""
import math
import os
import sys

import pytest

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench  # noqa: E402
from paper_2007_01045_b200.runtime import merge_timelines  # noqa: E402


def test_flops_per_sample_match_survey():
    assert bench.flops_per_sample(bench.MODELS["bert48"]) == pytest.approx(2.010e12, rel=1e-3)
    assert bench.flops_per_sample(bench.MODELS["vgg19"]) == pytest.approx(117.8e9, rel=1e-3)
    # GPT-2: 67,993,600 FLOP/token/layer x48 + head, x3 x1024 tokens (head at V = 50257)
    gpt = bench.flops_per_sample(bench.MODELS["gpt2-1.5b"])
    assert gpt == pytest.approx(3 * 1024 * (48 * 67_993_600 + 2 * 1600 * 50257), rel=1e-9)


@pytest.mark.parametrize("n", [1, 2, 4, 8])
def test_plans_cover_the_layers(n):
    for name, model in bench.MODELS.items():
        straight = bench.DEFAULTS[name]["straight"]
        plan = bench.make_plan(n, model["layers"], straight, model["kind"], sum(model.get("convs", [16])))
        gpus = [g for s in plan["stages"] for g in s["gpus"]]
        assert sorted(gpus) == list(range(n))
        assert plan["stages"][0]["layers"][0] == 0 and plan["stages"][-1]["layers"][1] == model["layers"]
        for a, b in zip(plan["stages"], plan["stages"][1:]):
            assert a["layers"][1] == b["layers"][0]
    vgg8 = bench.make_plan(8, 19, False, "vgg")
    assert [len(s["gpus"]) for s in vgg8["stages"]] == [6, 2]  # C3: conv r=6, FC r=2
    gpt8 = bench.make_plan(8, 48, True)
    assert [s["layers"] for s in gpt8["stages"]] == [[6 * k, 6 * k + 6] for k in range(8)]  # C4


def test_vgg_shapes_table():
    v = bench.vgg_shapes(bench.MODELS["vgg19"])
    assert len(v) == 19 and sum(x["conv"] for x in v) == 16
    assert v[15]["pool"] and v[16]["fin"] == 7 * 7 * 512 and v[18]["fout"] == 1000


def test_slice_profile_scales_by_replication():
    base = {"profile_batch_size": 8, "layers": [{"fwd_time_us": 10.0, "bwd_time_us": 20.0, "activation_bytes": 1,
                                                 "param_bytes": 1}] * 4}
    half = {"profile_batch_size": 4, "layers": [{"fwd_time_us": 6.0, "bwd_time_us": 11.0, "activation_bytes": 1,
                                                 "param_bytes": 1}] * 4}
    plan = {"stages": [{"layers": [0, 2], "gpus": [0]}, {"layers": [2, 4], "gpus": [1, 2]}]}
    p = bench.slice_profile({8: base, 4: half}, plan, 8)
    assert p["layers"][0]["fwd_time_us"] == 10.0
    assert p["layers"][3]["fwd_time_us"] == 12.0 and p["layers"][3]["bwd_time_us"] == 22.0  # slice time x r


def test_merge_timelines_aligns_ranks_and_computes_bubble():
    # two ranks, 2 stages (expanded 3), M = 2; rank 1's timer starts 1 ms later
    r0 = {"t0_ns": 0, "step_s": 0.010, "stage": 0,
          "blocks": [[0, 0, 0, 0.000, 0.001], [0, 1, 0, 0.001, 0.002], [0, 0, 1, 0.005, 0.007], [0, 1, 1, 0.007, 0.009],
                     [1, 0, 0, 0.001, 0.0012], [1, 1, 0, 0.002, 0.0022]]}
    r1 = {"t0_ns": 1_000_000, "step_s": 0.008, "stage": 1,
          "blocks": [[2, 0, 0, 0.0005, 0.0015], [2, 0, 1, 0.0015, 0.0035], [2, 1, 0, 0.0035, 0.0045],
                     [2, 1, 1, 0.0045, 0.0065]]}
    m = merge_timelines([r0, r1], 2, 2)
    assert len(m["blocks"]) == 2 * 2 * 3
    f = {(x, i, k): (s, e) for x, i, k, s, e in m["blocks"] if not math.isnan(s)}
    assert f[(2, 0, 0)] == pytest.approx((0.0015, 0.0025))  # shifted onto rank 0's timer
    assert m["latency"] == pytest.approx(0.010)  # first forward at 0 -> last rank done at 10 ms
    busy = (0.001 + 0.001 + 0.002 + 0.002) + (0.001 + 0.002 + 0.001 + 0.002)
    assert m["bubble"] == pytest.approx(1 - busy / (2 * 0.010))


def test_comm_stats_rates():
    """Split-Concat GB/s from send blocks and AllReduce bus bandwidth per block."""
    tl0 = {"stage": 0, "replication": 2, "allreduce_impl": "peer", "send_bytes": 8 << 20, "send_back_bytes": 0,
           "blocks": [[0, 0, 0, 0.0, 1.0], [1, 0, 0, 1.0, 1.0 + 0.01]],
           "allreduce": [[0, 2.0, 2.0 + 0.001, 100_000_000]]}
    tl1 = {"stage": 1, "replication": 1, "send_bytes": 0, "send_back_bytes": 4 << 20,
           "blocks": [[2, 0, 0, 1.1, 1.2], [1, 0, 1, 1.3, 1.3 + 0.004]], "allreduce": []}
    c = bench.comm_stats([tl0, tl1], {"bw_gbps": 800.0, "latency_us": 3.0})
    assert c["splitconcat"]["sends"] == 2
    assert c["splitconcat"]["gbps_median"] == pytest.approx(((8 << 20) / 0.01 + (4 << 20) / 0.004) / 2 / 1e9)
    ar = c["allreduce"]
    assert ar["impl"] == "peer" and ar["blocks"] == 1
    assert ar["busbw_gbps_median"] == pytest.approx(2 * 1 / 2 * 1e8 / 0.001 / 1e9)
    assert ar["frac_of_link"] == pytest.approx(ar["busbw_gbps_median"] / 800.0)


def test_planner_cpu_times_match_reference():
    """The CPU baseline's planner leg: the reference's plan() (oracle/_ref) and
    the new host planner give the same plan for the same request."""
    from oracle import refproc
    if not refproc.available():
        pytest.skip("oracle/_ref not built")
    prof = {"profile_batch_size": 8, "layers": [
        {"fwd_time_us": 100.0 + 7 * i, "bwd_time_us": 210.0, "activation_bytes": 1 << 23, "param_bytes": 50 << 20}
        for i in range(24)]}
    cl = bench.b200_cluster(4, 4.0)
    from paper_2007_01045_b200 import pipeplan
    plan = pipeplan.plan(prof, cl, 8)["plan"]
    out = bench.planner_cpu_times(prof, cl, 8, plan)
    assert out["identical_plan"] and out["identical_sim_latency"]
    assert out["reference_plan_s"] > 0 and out["ours_plan_par_s"] > 0


def test_plan_fixed_point_replans_on_slice_profiles(monkeypatch):
    """plan_fixed_point re-profiles at the chosen plan's slice sizes until
    the plan repeats (fake profiler: per-sample cost with a fixed overhead, so
    smaller slices are less efficient than the planner's ÷r assumes)."""
    calls = []

    def fake_profile(model, samples, reps=5):
        calls.append(samples)
        return {"profile_batch_size": samples, "layers": [
            {"fwd_time_us": 50.0 + 10.0 * samples, "bwd_time_us": 100.0 + 20.0 * samples,
             "activation_bytes": samples << 20, "param_bytes": 50 << 20} for _ in range(24)]}

    monkeypatch.setattr(bench, "profile_model", fake_profile)
    profiles = {8: fake_profile(None, 8)}
    plan, info = bench.plan_fixed_point({"layers": 24}, profiles, 8, bench.b200_cluster(4, 6.0), 8)
    assert info["fixed_point"]
    chosen = [[s["layers"], s["gpus"]] for s in plan["stages"]]
    # a proposal of some chain, or one of the planner's top-k runners-up
    assert any(it["stages"] == chosen for it in info["iterations"] + info["alternatives"])
    assert info["sim_latency_ms"] > 0
    # every chain starts from the full micro-batch or a replica slice of it
    assert {it["start_slice"] for it in info["iterations"]} <= {8, 4, 3, 2}
    assert info["iterations"][0]["start_slice"] == 8
    for st in plan["stages"]:
        assert -(-8 // len(st["gpus"])) in profiles


def test_plan_fixed_point_picks_the_self_consistent_best(monkeypatch):
    """When re-planning on a plan's own slice profile proposes a different
    plan (the ÷r model flatters small slices), the loop stops at the first
    repeat and runs the proposal with the lowest L evaluated on its OWN slice
    profile -- the L it reports."""
    from paper_2007_01045_b200 import pipeplan

    def fake_profile(model, samples, reps=5):
        # strongly sub-linear: a 1-sample slice costs 60% of an 8-sample one
        t = 100.0 * (0.55 + 0.45 * samples / 8)
        return {"profile_batch_size": samples, "layers": [
            {"fwd_time_us": t, "bwd_time_us": 2 * t, "activation_bytes": samples << 20, "param_bytes": 50 << 20}
            for _ in range(24)]}

    monkeypatch.setattr(bench, "profile_model", fake_profile)
    profiles = {8: fake_profile(None, 8)}
    cl = bench.b200_cluster(4, 180.0)
    plan, info = bench.plan_fixed_point({"layers": 24}, profiles, 8, cl, 8)
    sims = [it["own_profile_sim_ms"] for it in info["iterations"] + info["alternatives"]]
    assert info["sim_latency_ms"] == pytest.approx(min(sims))
    assert info["sim_latency_ms"] <= min(it["own_profile_sim_ms"] for it in info["iterations"])
    own = bench.slice_profile(profiles, plan, 8)
    assert pipeplan.simulate_plan(plan, own, cl, 8)["latency"] * 1e3 == pytest.approx(info["sim_latency_ms"])
    starts = {it["start_slice"] for it in info["iterations"]}
    assert all(sum(it["start_slice"] == st for it in info["iterations"]) <= 5 for st in starts)


def test_amoebanet_stand_in_shapes():
    """C5's AmoebaNet-36 stand-in: 36 profile layers, 3 resolution stages with
    growing channels (parameters grow, activations shrink with depth)."""
    m = bench.MODELS["amoebanet36"]
    v = bench.vgg_shapes(m)
    assert len(v) == m["layers"] == 36 and sum(x["conv"] for x in v) == 35
    assert [v[i]["cout"] for i in (0, 12, 24)] == [128, 256, 512]
    assert v[11]["pool"] and v[23]["pool"] and v[34]["pool"]
    assert v[35] == dict(conv=False, fin=16 * 16 * 512, fout=1000)
    from oracle.executor_ref import Model, vgg_layer
    om = Model.from_dict(m)
    for l in range(36):
        o = vgg_layer(om, l)
        if v[l]["conv"]:
            assert (o["h"], o["cin"], o["cout"], o["pool"]) == (v[l]["h"], v[l]["cin"], v[l]["cout"], v[l]["pool"])
        else:
            assert (o["fin"], o["fout"], o["relu"]) == (v[l]["fin"], v[l]["fout"], False)
