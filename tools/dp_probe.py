"""2-rank DP step probe (graph on/off) -- torchrun worker."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2007_01045_b200.runtime import Executor  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dist.init_process_group("gloo")
ex = Executor(dict(kind="mlp", layers=4, hidden=256), {"stages": [{"layers": [0, 4], "gpus": [0, 1]}]}, 4, 24,
              rank=rank, world=world)
print(rank, "created", flush=True)
for i in range(3):
    print(rank, "step", i, ex.step(), flush=True)
ex.close()
print(rank, "done", flush=True)
