"""Wall time of Executor.step() with device-generated vs pinned-host inputs."""
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2007_01045_b200.runtime import Executor  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "vgg19"
model = bench.MODELS[name]
d = bench.DEFAULTS[name]
M, sl = d["micro_batches"], d["slice"]
gbs = M * sl
plan = bench.make_plan(1, model["layers"], d["straight"], model["kind"])
ex = Executor(model, plan, M, gbs, rank=0, world=1, device=0)
inp, tgt = bench.host_batches(model, plan, 0, M, gbs // M, 1234)
for _ in range(3):
    ex.step()
    ex.step(inp, tgt)
torch.cuda.synchronize()
for label, args in (("device", ()), ("host", (inp, tgt))):
    t = time.perf_counter()
    for _ in range(5):
        ex.step(*args)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t) / 5
    print(f"{label}: {dt * 1e3:.2f} ms/step  ({gbs / dt:.0f} samples/s)  inp {inp.numel() * inp.element_size() / 1e6:.1f} MB "
          f"pinned={inp.is_pinned()}")
t = time.perf_counter()
for _ in range(5):
    x = torch.empty_like(inp, device="cuda")
    x.copy_(inp, non_blocking=True)
torch.cuda.synchronize()
print(f"raw H2D of the step's inputs: {(time.perf_counter() - t) / 5 * 1e3:.2f} ms")
ex.close()
