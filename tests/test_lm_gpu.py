"""GPT language-model end kernels (lm.cu) vs the oracle's token generator and
plain torch fp32 references, plus the LM executor step vs the CPU oracle."""
import numpy as np
import pytest
import torch

from paper_2007_01045_b200 import kernels as K

pytestmark = pytest.mark.gpu


def _rand(*shape, dev, scale=1.0, dtype=torch.bfloat16, seed=0):
    g = torch.Generator(device="cpu").manual_seed(seed)
    return ((torch.rand(*shape, generator=g) * 2 - 1) * scale).to(dtype).to(dev)


def test_fill_tokens_bit_exact_with_oracle(cuda):
    from oracle.executor_ref import Model, lm_tokens
    m = Model.from_dict(dict(kind="gpt", layers=1, hidden=64, heads=1, seq=128, vocab=50304))
    tok, tgt = lm_tokens(m, 1234, 5, 3)  # samples 5..7
    out = torch.empty(tok.size, dtype=torch.int32, device=cuda)
    K.fill_tokens(out, tok.size, 1234, 1, 5 * 128, 50304)
    assert np.array_equal(out.cpu().numpy(), tok)
    K.fill_tokens(out, tok.size, 1234, 2, 5 * 128, 50304)
    assert np.array_equal(out.cpu().numpy(), tgt)


@pytest.mark.parametrize("rows,seq,h,v", [(256, 128, 256, 1000), (2048, 1024, 1600, 50304)])
def test_embedding_fwd_bwd(cuda, rows, seq, h, v):
    g = torch.Generator(device="cpu").manual_seed(3)
    tok = torch.randint(0, v, (rows,), generator=g, dtype=torch.int32).to(cuda)
    tok[:16] = 7  # repeated ids: the backward must add, not overwrite
    wte = _rand(v, h, dev=cuda, seed=1, scale=0.1)
    wpe = _rand(seq, h, dev=cuda, seed=2, scale=0.1)
    x = torch.empty(rows, h, dtype=torch.bfloat16, device=cuda)
    K.embed_fwd(tok, wte, wpe, x, rows, seq, h)
    pos = torch.arange(rows, device=cuda) % seq
    ref = (wte[tok.long()].float() + wpe[pos].float()).bfloat16()
    assert torch.equal(x, ref)
    dx = _rand(rows, h, dev=cuda, seed=4)
    gwte = torch.zeros(v, h, device=cuda)
    gwpe = torch.zeros(seq, h, device=cuda)
    K.embed_bwd(tok, dx, gwte, gwpe, rows, seq, h)
    rte = torch.zeros(v, h, device=cuda).index_add_(0, tok.long(), dx.float())
    rpe = torch.zeros(seq, h, device=cuda).index_add_(0, pos, dx.float())
    torch.cuda.synchronize()
    assert torch.allclose(gwte, rte, rtol=1e-5, atol=1e-5)
    assert torch.allclose(gwpe, rpe, rtol=1e-5, atol=1e-5)


@pytest.mark.parametrize("rows,v", [(64, 1000), (300, 50304), (8, 8)])
def test_cross_entropy_fwd_bwd(cuda, rows, v):
    logits = _rand(rows, v, dev=cuda, seed=5, scale=8.0)
    g = torch.Generator(device="cpu").manual_seed(6)
    tgt = torch.randint(0, v, (rows,), generator=g, dtype=torch.int32).to(cuda)
    lf = logits.float().requires_grad_(True)
    ref = torch.nn.functional.cross_entropy(lf, tgt.long(), reduction="sum")
    (dref,) = torch.autograd.grad(ref, lf)
    scale = 1.0 / (rows * 4)
    acc = torch.zeros(1, device=cuda)
    work = logits.clone()
    K.cross_entropy(work, tgt, acc, rows, v, scale)
    torch.cuda.synchronize()
    assert abs(acc.item() - ref.item()) <= 1e-4 * abs(ref.item()) + 1e-3
    err = (work.float() - dref * scale).abs().max().item()
    assert err <= 0.01 * (dref * scale).abs().max().item()


@pytest.mark.parametrize("rows,v", [(64, 1001), (300, 50257), (8, 1)])
def test_cross_entropy_padded_vocab(cuda, rows, v):
    """Rows of stride ld = v rounded up to 8 (C4's 50257 stored as 50264):
    the padding columns hold garbage that must not enter the softmax and get
    a zero gradient."""
    ld = (v + 7) // 8 * 8
    logits = _rand(rows, ld, dev=cuda, seed=7, scale=8.0)
    logits[:, v:] = 30.0  # would dominate the softmax if not masked
    g = torch.Generator(device="cpu").manual_seed(8)
    tgt = torch.randint(0, v, (rows,), generator=g, dtype=torch.int32).to(cuda)
    lf = logits[:, :v].float().requires_grad_(True)
    ref = torch.nn.functional.cross_entropy(lf, tgt.long(), reduction="sum")
    (dref,) = torch.autograd.grad(ref, lf)
    scale = 1.0 / rows
    acc = torch.zeros(1, device=cuda)
    work = logits.clone()
    K.cross_entropy_padded(work, tgt, acc, rows, v, ld, scale)
    torch.cuda.synchronize()
    assert abs(acc.item() - ref.item()) <= 1e-4 * abs(ref.item()) + 1e-3
    err = (work[:, :v].float() - dref * scale).abs().max().item()
    assert err <= 0.01 * (dref * scale).abs().max().item() + 1e-6
    assert bool((work[:, v:] == 0).all())


LM = dict(kind="gpt", layers=2, hidden=256, heads=4, ffn=1024, seq=128, vocab=1000)
# vocabulary not a multiple of 8 (padded projection rows, masked logits)
LM_ODD = dict(kind="gpt", layers=2, hidden=256, heads=4, ffn=1024, seq=128, vocab=1001)


def _check_lm_tensors(ex, emu, exact, stage_first, stage_last):
    from parity_util import EMU_GRAD_RTOL, FP64_GRAD_RTOL, rel_fro
    names = ([("emb", "wte"), ("emb", "wpe")] if stage_first else []) + \
        ([("head", "Wout"), ("head", "lnf_g"), ("head", "lnf_b")] if stage_last else [])
    for owner, name in names:
        want = emu.grads[(owner, name)]
        got = ex.read(owner, name, want.size, grad=True)
        e = rel_fro(got, want)
        assert e < EMU_GRAD_RTOL, f"{owner}.{name}: grad rel err vs bf16 oracle {e:.4g}"
        assert rel_fro(got, exact.grads[(owner, name)]) < FP64_GRAD_RTOL


@pytest.mark.parametrize("schedule,recompute,model", [("dapple", False, "LM"), ("gpipe", True, "LM"),
                                                      ("dapple", False, "LM_ODD")])
def test_lm_single_gpu_step_matches_oracle(cuda, schedule, recompute, model):
    from oracle.executor_ref import full_batch_step
    from parity_util import check_grads, check_loss
    from paper_2007_01045_b200.runtime import Executor
    plan = {"stages": [{"layers": [0, 2], "gpus": [0], "replication": 1}]}
    model = {"LM": LM, "LM_ODD": LM_ODD}[model]
    exact = full_batch_step(model, 8)
    emu = full_batch_step(model, 8, bf16=True)
    ex = Executor(model, plan, 4, 8, lr=1e-3, apply=False, schedule=schedule, recompute=recompute)
    loss = ex.step()
    assert abs(loss - np.log(model["vocab"])) < 1.0  # near-uniform predictions at init
    check_loss(loss, emu, exact)
    check_grads(ex, emu, exact, range(2), "gpt", 2)
    _check_lm_tensors(ex, emu, exact, True, True)
    ex.close()


def test_lm_profile_and_host_tokens(cuda):
    """Host token ids through the public step (e2e path) give the same loss as
    device-generated ones; the profiler folds embedding/head into the end layers."""
    from paper_2007_01045_b200.runtime import Executor
    plan = {"stages": [{"layers": [0, 2], "gpus": [0], "replication": 1}]}
    ex = Executor(LM, plan, 2, 4, lr=0.0, apply=False)
    l_dev = ex.step()
    rows = 2 * 128
    tok = torch.empty(2, rows, dtype=torch.int32, device=cuda)
    tgt = torch.empty(2, rows, dtype=torch.int32, device=cuda)
    for i in range(2):
        K.fill_tokens(tok[i], rows, 1234, 1, i * rows, 1000)
        K.fill_tokens(tgt[i], rows, 1234, 2, i * rows, 1000)
    torch.cuda.synchronize()
    l_host = ex.step(tok.cpu().pin_memory(), tgt.cpu().pin_memory())
    assert abs(l_host - l_dev) <= 1e-6 * abs(l_dev)
    prof = ex.layer_profile(2)
    h, v = 256, 1000
    base = (12 * h * h + 13 * h) * 4
    assert prof["layers"][0]["param_bytes"] == base + (v * h + 128 * h) * 4
    assert prof["layers"][1]["param_bytes"] == base + (2 * h + v * h) * 4
    ex.close()


def test_lm_causal_split_attention_step(cuda):
    """seq 512: causal query tiles with >= 4 key tiles run as two CTAs whose
    partials merge in the second to finish (attention.cu, fwd_part / fwd_flags).
    The step matches the oracle and repeats (the tickets re-arm)."""
    from oracle.executor_ref import full_batch_step
    from parity_util import check_grads, check_loss
    from paper_2007_01045_b200.runtime import Executor
    lm = dict(LM, seq=512)
    plan = {"stages": [{"layers": [0, 2], "gpus": [0], "replication": 1}]}
    exact = full_batch_step(lm, 4)
    emu = full_batch_step(lm, 4, bf16=True)
    ex = Executor(lm, plan, 4, 4, lr=0.0, apply=False)
    loss = ex.step()
    check_loss(loss, emu, exact)
    check_grads(ex, emu, exact, range(2), "gpt", 2)
    losses = [ex.step() for _ in range(3)]
    assert all(abs(l - loss) <= 1e-6 * abs(loss) for l in losses), (loss, losses)  # CE sums with atomics
    ex.close()
