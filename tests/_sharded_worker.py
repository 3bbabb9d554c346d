"""torchrun worker for tests/test_sharding_gpu.py::test_two_ranks_raise_the_same_violation:
two gloo ranks on one GPU, a |c| > 1 sample in rank 1's shard; each rank
prints the AmplitudeBoundError it raised."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
import paper_2108_07126_b200 as sp  # noqa: E402
from cases import random_inputs  # noqa: E402
from paper_2108_07126_b200.sharding import (equiprop_sharded_device, partition,  # noqa: E402
                                            shard_rows)

dist.init_process_group("gloo")
rank, world = dist.get_rank(), dist.get_world_size()
torch.cuda.set_device(0)
h0, hs, values, dt = random_inputs(4, 2, 100, 23)
values = values.copy()
values[70, 0] = -1.25
ctx = sp.create(device=0)
ctx.set_hamiltonian(sp.ControlSystem(h0, hs))
a, b = partition(100, world)[rank]
lo, hi = shard_rows("midpoint", a, b)
local = torch.from_numpy(np.ascontiguousarray(values[lo:hi])).cuda()
try:
    equiprop_sharded_device(ctx, local, dt, 100)
    print(f"RANK{rank}:no error", flush=True)
except sp.AmplitudeBoundError as exc:
    print(f"RANK{rank}:{exc}", flush=True)
dist.barrier()
dist.destroy_process_group()
