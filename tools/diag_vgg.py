"""Per-layer gradient error of the device VGG step vs the bf16 oracle."""
import json
import sys

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import torch  # noqa: E402,F401

from oracle.executor_ref import full_batch_step  # noqa: E402
from parity_util import rel_fro  # noqa: E402
from paper_2007_01045_b200.runtime import Executor  # noqa: E402

m = json.loads(sys.argv[1]) if len(sys.argv) > 1 else dict(kind="vgg", layers=19, image=64, width=64, fc=128,
                                                           classes=16)
gbs = int(sys.argv[2]) if len(sys.argv) > 2 else 4
M = int(sys.argv[3]) if len(sys.argv) > 3 else 1
emu = full_batch_step(m, gbs, bf16=True)
plan = {"stages": [{"layers": [0, 19], "gpus": [0], "replication": 1}]}
ex = Executor(m, plan, M, gbs, apply=False)
loss = ex.step()
print("loss", loss, "oracle", emu.loss)
for l in range(19):
    out = []
    for name in ("W", "b"):
        got = ex.read(l, name, emu.grads[(l, name)].size, grad=True)
        out.append(f"{name} {rel_fro(got, emu.grads[(l, name)]):.4f}")
    print(l, *out)
ex.close()
