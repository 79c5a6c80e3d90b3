"""Executor API robustness: host buffers (pinned, rotating, pageable), input
validation, and plan / phi validation before any stream program is built."""
import pytest

pytestmark = pytest.mark.gpu

BERT = dict(kind="bert", layers=2, hidden=256, heads=4, ffn=1024, seq=128)
LM = dict(kind="gpt", layers=2, hidden=256, heads=4, ffn=1024, seq=128, vocab=1000)
ONE = {"stages": [{"layers": [0, 2], "gpus": [0], "replication": 1}]}


def _host_data(ex, model, M, gbs, seed, pinned=True):
    """The executor's own synthetic inputs / targets, copied to host memory."""
    import torch
    from paper_2007_01045_b200 import kernels
    rows = gbs // M * model["seq"]
    if model.get("vocab"):
        x = torch.empty((M, rows), dtype=torch.int32, device="cuda")
        t = torch.empty((M, rows), dtype=torch.int32, device="cuda")
        for i in range(M):
            kernels.fill_tokens(x[i], rows, seed, 1, i * rows, model["vocab"])
            kernels.fill_tokens(t[i], rows, seed, 2, i * rows, model["vocab"])
    else:
        h = model["hidden"]
        x = torch.empty((M, rows, h), dtype=torch.bfloat16, device="cuda")
        t = torch.empty((M, rows, h), dtype=torch.bfloat16, device="cuda")
        for i in range(M):
            kernels.fill_uniform_bf16(x[i], rows * h, seed, 1, i * rows * h)
            kernels.fill_uniform_bf16(t[i], rows * h, seed, 2, i * rows * h)
    torch.cuda.synchronize()
    x, t = x.cpu(), t.cpu()
    return (x.pin_memory(), t.pin_memory()) if pinned else (x, t)


@pytest.mark.parametrize("model", [BERT, LM])
def test_rotating_and_pageable_host_buffers(cuda, model):
    """A loader handing in a fresh buffer every step re-points the captured
    copy nodes instead of re-capturing: the graph count stays at one per
    (flag bank, host-data mode) and every buffer gives the device-data loss."""
    from paper_2007_01045_b200.runtime import Executor
    M, gbs = 2, 4
    ex_dev = Executor(model, ONE, M, gbs, apply=False)
    ref = ex_dev.step()
    ex_dev.close()
    ex = Executor(model, ONE, M, gbs, apply=False)
    bufs = [_host_data(ex, model, M, gbs, 1234) for _ in range(3)]
    losses = []
    for k in range(6):  # three rotating pinned buffer pairs, both flag banks
        losses.append(ex.step(*bufs[k % 3]))
    assert ex.graphs() == 2, ex.graphs()
    pageable = _host_data(ex, model, M, gbs, 1234, pinned=False)
    assert not pageable[0].is_pinned()
    losses.append(ex.step(*pageable))
    losses.append(ex.step(*pageable))
    assert ex.graphs() == 2
    ex.close()
    # apply=False: gradients accumulate but the weights and so the loss do not move
    for lo in losses:
        assert abs(lo - ref) <= 1e-6 * abs(ref), (lo, ref)


def test_host_inputs_are_validated(cuda):
    import torch
    from paper_2007_01045_b200.runtime import Executor
    ex = Executor(LM, ONE, 2, 4, apply=False)
    x, t = _host_data(ex, LM, 2, 4, 1234)
    with pytest.raises(ValueError, match="bytes"):
        ex.step(x[:1], t)
    with pytest.raises(TypeError, match="dtype"):
        ex.step(x.to(torch.int64), t)
    bad = t.clone()
    bad[0, 0] = 1000  # == vocab
    with pytest.raises(ValueError, match="ids"):
        ex.step(x, bad)
    strided = torch.empty((x.shape[1], x.shape[0]), dtype=x.dtype).t()
    strided.copy_(x)
    with pytest.raises(ValueError, match="contiguous"):
        ex.step(strided, t)
    ex.step(x, t)  # and the valid call still works
    ex.close()


@pytest.mark.parametrize("plan,msg", [
    ({"stages": [{"layers": [0, 1], "gpus": [0]}, {"layers": [1, 2], "gpus": [0]}], "phi": [1, 1]}, "more than one"),
    ({"stages": [{"layers": [0, 2], "gpus": [-1]}]}, "negative"),
    ({"stages": [{"layers": [0, 1], "gpus": [0]}, {"layers": [1, 2], "gpus": [1]}], "phi": [1, 2]},
     "non-increasing"),
    ({"stages": [{"layers": [0, 1], "gpus": [0]}, {"layers": [1, 2], "gpus": [1]}],
      "phi_expanded": [2, 2, 2]}, "topmost"),
])
def test_executor_rejects_invalid_plans(cuda, plan, msg):
    """The executor refuses plans whose flag waits could never be satisfied
    (reference PipelinePlan::validate / check_phi semantics) instead of
    deadlocking the ranks."""
    from paper_2007_01045_b200.runtime import Executor
    with pytest.raises(RuntimeError, match=msg):
        Executor(BERT, plan, 4, 8, rank=0, world=2, apply=False)
