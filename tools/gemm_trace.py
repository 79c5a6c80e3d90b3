"""Phase breakdown of one GEMM launch from the kernel's %globaltimer trace
(GemmDesc::trace): per CTA entry / prologue / first TMA / first MMA / last
commit / epilogue start / epilogue end / exit, in us relative to the
earliest entry.  python tools/gemm_trace.py o|ffn1|wgrad_gpt [--1sm]"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2007_01045_b200 import kernels as K  # noqa: E402

dev = torch.device("cuda:0")
bf = torch.bfloat16
which = sys.argv[1]
one = "--1sm" in sys.argv
shapes = {"o": (4096, 1024, 1024, "fwd", K.EPI_BIAS | K.EPI_RESID), "ffn1": (4096, 4096, 1024, "fwd", K.EPI_BIAS | K.EPI_GELU | K.EPI_AUX_OUT),
          "qkv": (4096, 3072, 1024, "fwd", K.EPI_BIAS), "ffn2": (4096, 1024, 4096, "fwd", K.EPI_BIAS | K.EPI_RESID),
          "plain": (4096, 1024, 1024, "fwd", 0), "wgrad_gpt": (1600, 6400, 1024, "wgrad", 0),
          "wgrad_o": (1024, 1024, 4096, "wgrad", 0), "big": (8192, 8192, 8192, "fwd", 0),
          "gpt_ffn2": (1024, 1600, 6400, "fwd", K.EPI_BIAS | K.EPI_RESID), "gpt_ffn2_plain": (1024, 1600, 6400, "fwd", 0)}
M, N, Kd, kind, epi = shapes[which]
W = 64  # trace words per CTA (gemm_tcgen05.cu kTraceWords)
tr = torch.zeros(148 * W, dtype=torch.int64, device=dev)
if kind == "fwd":
    A = torch.randn(M, Kd, device=dev).to(bf); B = torch.randn(N, Kd, device=dev).to(bf)
    C = torch.empty(M, N, device=dev, dtype=bf); X = torch.empty(M, N, device=dev, dtype=bf)
    R = torch.randn(M, N, device=dev).to(bf); bias = torch.zeros(N, device=dev)
    f = lambda t: K.gemm(A, B, C, M, N, Kd, lda=Kd, ldb=Kd, ldc=N, epi=epi, bias=bias, resid=R if epi & K.EPI_RESID else None,
                         aux_out=X if epi & K.EPI_AUX_OUT else None, force_1sm=one, trace=t)
else:
    A = torch.randn(Kd, M, device=dev).to(bf); B = torch.randn(Kd, N, device=dev).to(bf)
    C = torch.zeros(M, N, device=dev)
    f = lambda t: K.gemm(A, B, C, M, N, Kd, lda=M, ldb=N, ldc=N, a_mn_major=True, b_mn_major=True,
                         epi=K.EPI_OUT_F32_ACC, force_1sm=one, trace=t)
for _ in range(5):
    f(None)
for _ in range(3):
    f(tr)
torch.cuda.synchronize()
full = tr.view(148, W).cpu().numpy().astype("float64")
t = full[:, :16]
used = t[:, 0] > 0
t = t[used]
full = full[used]
r = t - t[:, :1]  # cycles since this CTA's entry
names = ["entry", "prologue", "first_tma", "first_mma", "last_commit", "epi_start", "epi_end", "exit",
         "c0_tmem", "c0_epi_done", "c0_before_xwait", "c0_after_xwait", "c1_tmem", "c1_epi_done", "c1_before_xwait", "c1_after_xwait"]
import numpy as np  # noqa: E402
print(f"{which} {M}x{N}x{Kd} ctas={used.sum()} 1sm={one} (cycles since CTA entry)")
for i, n in enumerate(names):
    sel = t[:, i] > 0
    if not sel.any():
        continue
    nz = r[sel, i]
    print(f"  {n:12s} min {nz.min():8.0f}  median {np.median(nz):8.0f}  max {nz.max():8.0f}  (n={len(nz)})")

# per-tile timeline: SM clock -> ns via each CTA's entry / exit globaltimer
clk = (full[:, 7] - full[:, 0]) / np.maximum(full[:, 62] - full[:, 63], 1)  # cycles per ns
t0 = full[:, 63].min()
print(f"  ring stages {int(full[0, 61])}; SM clock ~{np.median(clk):.2f} GHz; kernel span {(full[:, 62].max() - t0) / 1e3:.2f} us")
rows = []
for c in range(full.shape[0]):
    ent = (full[c, 63] - t0) / 1e3
    tiles = []
    for j in range(6):
        v = full[c, 16 + 4 * j:20 + 4 * j]
        if v[0] <= 0:
            break
        tiles.append([ent + (x - full[c, 0]) / clk[c] / 1e3 if x > 0 else float("nan") for x in v])
    rows.append((ent, tiles, ent + (full[c, 7] - full[c, 0]) / clk[c] / 1e3))
print("  per tile (us from the first CTA entry): mma_start-mma_end | epi_start-epi_end")
for c in list(range(0, len(rows), max(1, len(rows) // 8))):
    ent, tiles, ex = rows[c]
    desc = "  ".join(f"[{a:6.2f}-{b:6.2f}|{e0:6.2f}-{e1:6.2f}]" for a, b, e0, e1 in tiles)
    print(f"  cta {c:3d} entry {ent:6.2f} exit {ex:6.2f}: {desc}")
mma = [b - a for _, tiles, _ in rows for a, b, _, _ in tiles]
epi = [e1 - e0 for _, tiles, _ in rows for _, _, e0, e1 in tiles if e1 == e1]
gap = [tiles[j + 1][0] - tiles[j][1] for _, tiles, _ in rows for j in range(len(tiles) - 1)]
kb = -(-Kd // 64)
print(f"  cycles per 64-wide k-block: median {np.median(mma) * 1e3 * np.median(clk) / kb:.0f} (MMA floor 512 for 256-wide tiles)")
print(f"  mma span per tile: median {np.median(mma):.2f} us; epilogue per tile: median {np.median(epi):.2f} us;"
      f" gap mma_end -> next mma_start: median {np.median(gap) if gap else 0:.2f} us")

steps = ["tmem_ld", "wait_ld", "wait_store_read", "stage_sts", "fence", "store_issue"]
for j in range(2):
    sl = full[:, 40 + 8 * j:46 + 8 * j]
    ok = sl[:, 0] > 0
    if ok.any():
        d = np.diff(sl[ok], axis=1)
        print(f"  chunk {j} of warp 4 (cycles): " + ", ".join(f"{steps[k + 1]} {np.median(d[:, k]):.0f}" for k in range(5)))
    if j == 0:
        nxt = full[:, 48]
        ok2 = (nxt > 0) & (sl[:, 5] > 0)
        if ok2.any():
            print(f"  chunk 0 store issued -> chunk 1 start: {np.median(nxt[ok2] - sl[ok2, 5]):.0f} cycles")
