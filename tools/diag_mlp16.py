import sys
sys.path.insert(0, "."); sys.path.insert(0, "tests")
from oracle.executor_ref import full_batch_step  # noqa
from paper_2007_01045_b200.runtime import Executor  # noqa
from parity_util import rel_fro  # noqa
model = dict(kind="mlp", layers=16, hidden=1024)
emu = full_batch_step(model, 64, bf16=True)
ex = Executor(model, {"stages": [{"layers": [0, 16], "gpus": [0]}]}, 8, 64, apply=False)
print("loss", ex.step(), emu.loss)
for l in range(16):
    g = ex.read(l, "W", 1024 * 1024, grad=True)
    b = ex.read(l, "b", 1024, grad=True)
    print(l, round(rel_fro(g, emu.grads[(l, "W")]), 4), round(rel_fro(b, emu.grads[(l, "b")]), 4))
