"""Multi-GPU executor parity (straight pipelines, uneven replication with
Split-Concat, replica AllReduce) -- runs torchrun over the visible GPUs."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))

MLP = dict(kind="mlp", layers=4, hidden=256)
BERT = dict(kind="bert", layers=4, hidden=256, heads=4, ffn=1024, seq=128)

CASES = [
    (2, MLP, {"stages": [{"layers": [0, 2], "gpus": [0]}, {"layers": [2, 4], "gpus": [1]}]}, 4, 24),
    (2, MLP, {"stages": [{"layers": [0, 4], "gpus": [0, 1]}]}, 4, 24),
    (2, BERT, {"stages": [{"layers": [0, 1], "gpus": [0]}, {"layers": [1, 4], "gpus": [1]}]}, 4, 8),
    (4, MLP, {"stages": [{"layers": [0, 3], "gpus": [0, 1, 2]}, {"layers": [3, 4], "gpus": [3]}]}, 4, 24),
    (4, MLP, {"stages": [{"layers": [0, 1], "gpus": [0]}, {"layers": [1, 4], "gpus": [1, 2, 3]}]}, 4, 24),
    (4, BERT, {"stages": [{"layers": [0, 2], "gpus": [0, 1]}, {"layers": [2, 4], "gpus": [2, 3]}]}, 4, 16),
    (4, BERT, {"stages": [{"layers": [0, 1], "gpus": [0]}, {"layers": [1, 2], "gpus": [1]},
                          {"layers": [2, 3], "gpus": [2]}, {"layers": [3, 4], "gpus": [3]}]}, 8, 8),
]
# replicas that do not divide the micro-batch (planner plans such as [0,6)x1 [6,48)x7 at mb=8)
CASES += [
    (2, MLP, {"stages": [{"layers": [0, 4], "gpus": [0, 1]}]}, 4, 28),
    (4, MLP, {"stages": [{"layers": [0, 3], "gpus": [0, 1, 2]}, {"layers": [3, 4], "gpus": [3]}]}, 4, 28),
    (4, BERT, {"stages": [{"layers": [0, 1], "gpus": [0]}, {"layers": [1, 4], "gpus": [1, 2, 3]}]}, 2, 8),
]
# GPT language model (embedding on stage 0, LN_f + vocab projection + CE on the last stage)
LMGPT = dict(kind="gpt", layers=4, hidden=256, heads=4, ffn=1024, seq=128, vocab=1000)
CASES += [
    (2, LMGPT, {"stages": [{"layers": [0, 2], "gpus": [0]}, {"layers": [2, 4], "gpus": [1]}]}, 4, 8),
    (4, LMGPT, {"stages": [{"layers": [0, 2], "gpus": [0, 1]}, {"layers": [2, 4], "gpus": [2, 3]}]}, 4, 16),
]
# VGG-19 (C3 shape): uneven conv / FC replication, Split-Concat of the pooled features
VGGS = dict(kind="vgg", layers=19, image=32, width=8, fc=32, classes=16)
CASES += [
    (2, VGGS, {"stages": [{"layers": [0, 10], "gpus": [0]}, {"layers": [10, 19], "gpus": [1]}]}, 2, 8),
    (4, VGGS, {"stages": [{"layers": [0, 16], "gpus": [0, 1, 2]}, {"layers": [16, 19], "gpus": [3]}]}, 2, 12),
]
# eight ranks: C2's structure (2 stages x 4 replicas: Split-Concat 4 -> 4, a
# 4-way replica AllReduce) and C4's (a straight 8-stage LM pipeline)
C2_8 = {"stages": [{"layers": [0, 2], "gpus": [0, 1, 2, 3]}, {"layers": [2, 4], "gpus": [4, 5, 6, 7]}]}
LMGPT8 = dict(LMGPT, layers=8)
C4_8 = {"stages": [{"layers": [k, k + 1], "gpus": [k]} for k in range(8)]}
CASES8 = [(8, BERT, C2_8, 4, 32), (8, LMGPT8, C4_8, 8, 8)]
CASES += CASES8
TWO = {"stages": [{"layers": [0, 2], "gpus": [0]}, {"layers": [2, 4], "gpus": [1]}]}
# GPipe / re-computation on the device (the schedules of the paper's Table VI)
SCHED_CASES = [
    (2, VGGS, {"stages": [{"layers": [0, 12], "gpus": [0]}, {"layers": [12, 19], "gpus": [1]}]}, 4, 8, "gpipe", True),
    (2, LMGPT, TWO, 4, 8, "dapple", True),
    (4, LMGPT, {"stages": [{"layers": [0, 1], "gpus": [0]}, {"layers": [1, 4], "gpus": [1, 2, 3]}]}, 2, 8,
     "dapple", False),
    (2, BERT, TWO, 4, 8, "gpipe", False),
    (2, MLP, TWO, 4, 24, "dapple", True),
    (2, BERT, TWO, 4, 8, "gpipe", True),
    (4, BERT, {"stages": [{"layers": [0, 2], "gpus": [0, 1]}, {"layers": [2, 4], "gpus": [2, 3]}]}, 4, 16,
     "dapple", True),
]


def _gpus():
    try:
        import torch
        return torch.cuda.device_count()
    except Exception:
        return 0


@pytest.mark.parametrize("n,model,plan,M,gbs", CASES)
def test_multi_gpu_step_matches_oracle(n, model, plan, M, gbs):
    if _gpus() < n:
        pytest.skip(f"needs {n} GPUs")
    spec = json.dumps({"model": model, "plan": plan, "M": M, "gbs": gbs})
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", "--master-port=29517", os.path.join(HERE, "mgpu_worker.py"), spec]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    print(r.stdout[-4000:])
    assert r.returncode == 0, r.stderr[-4000:]


@pytest.mark.parametrize("n,model,plan,M,gbs,schedule,recompute", SCHED_CASES)
def test_multi_gpu_schedules_match_oracle(n, model, plan, M, gbs, schedule, recompute):
    if _gpus() < n:
        pytest.skip(f"needs {n} GPUs")
    spec = json.dumps({"model": model, "plan": plan, "M": M, "gbs": gbs, "schedule": schedule,
                       "recompute": recompute})
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", "--master-port=29518", os.path.join(HERE, "mgpu_worker.py"), spec]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    print(r.stdout[-4000:])
    assert r.returncode == 0, r.stderr[-4000:]
