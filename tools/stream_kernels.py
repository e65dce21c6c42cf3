"""Drive the streaming kernels at C4 and C5 sizes for an ncu metrics capture:
device noise (K x H FP64 write) and the MPPI softmax partial (cost + noise rows
read) -- tools/stream_kernels.py; numbers in profiles/r1_stream_kernels.json."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2509_16079_b200 import config  # noqa: E402
from paper_2509_16079_b200.device import DevicePlan, noise_philox  # noqa: E402

torch.cuda.set_device(0)
dev = torch.device("cuda")
v = config.VpmConfig(particle_cap=512)
ip, fp = config.pack_params(v, config.GliderParams())
plan = DevicePlan(ip, fp)
for K, H in ((4096, 50), (16384, 50), (65536, 50)):
    noise = torch.empty((K, H), dtype=torch.float64, device=dev)
    for _ in range(3):
        noise_philox(3, 0, noise)
    cost = torch.as_tensor(np.random.default_rng(0).uniform(0, 3, K + 1), device=dev)
    us = torch.full((H,), -6.0, dtype=torch.float64, device=dev)
    for _ in range(3):
        plan.mppi_partial(cost, us, noise, 2.0, 50.0)  # lambda 50: every row carries weight
torch.cuda.synchronize()
print("ok")
