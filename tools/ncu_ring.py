"""Small driver for ncu: single-device ring allreduce (virtual ranks, p=4,
2^24 values per member, rate 8) -- the decompress-add-recompress (DAR) step
kernels the ring uses, in isolation."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2409_02423_b200 import CodecSpec  # noqa: E402
from paper_2409_02423_b200 import collectives as K  # noqa: E402
from paper_2409_02423_b200.comm_path import CommPath  # noqa: E402
from paper_2409_02423_b200.netsim import SimClock, Topology  # noqa: E402

torch.cuda.set_device(0)
p, n = 4, 1 << 24
xs = [torch.randn(n, device="cuda") * 1e-3 for _ in range(p)]
clock = SimClock(Topology.b200_box(8))
for _ in range(2):
    K.allreduce(clock, K.Communicator(list(range(p))), xs, CodecSpec.fixed_rate(8), CommPath.DpAllReduce)
torch.cuda.synchronize()
print("ok", [round(e.duration_s * 1e6, 1) for e in clock.trace()])
