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
    # GPT-2: 67,993,600 FLOP/token/layer x48 + head, x3 x1024 tokens (head at V = 50304)
    gpt = bench.flops_per_sample(bench.MODELS["gpt2-1.5b"])
    assert gpt == pytest.approx(3 * 1024 * (48 * 67_993_600 + 2 * 1600 * 50304), rel=1e-9)


@pytest.mark.parametrize("n", [1, 2, 4, 8])
def test_plans_cover_the_layers(n):
    for name, model in bench.MODELS.items():
        straight = bench.DEFAULTS[name]["straight"]
        plan = bench.make_plan(n, model["layers"], straight, model["kind"])
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
