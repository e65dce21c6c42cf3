"""Warm in-stream device time of the streaming kernels (tuning tool, not product):
the MPPI softmax partial and the device-noise kernel, 50 launches queued back to
back behind a spin kernel under CUDA events (no host launch gaps), inputs L2-resident
as inside an iteration.  Prints one JSON line per (kernel, rows)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2509_16079_b200 import config  # noqa: E402
from paper_2509_16079_b200.device import DevicePlan, mppi_combine, noise_philox  # noqa: E402

torch.cuda.set_device(0)
dev = torch.device("cuda")
v = config.VpmConfig(particle_cap=512)
ip, fp = config.pack_params(v, config.GliderParams())
plan = DevicePlan(ip, fp)
H, REPS = 50, 50


def queued_time(fn):
    """Per-launch device time of REPS back-to-back launches: a spin kernel holds the
    stream while the host enqueues them, so no host launch gap enters the events."""
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3):
            fn(s)
        torch.cuda.synchronize()
        best = float("inf")
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda._sleep(20_000_000)  # ~10 ms of spinning
            e0.record(s)
            for _ in range(REPS):
                fn(s)
            e1.record(s)
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1) * 1e3 / REPS)
    return best


for K in (256, 512, 4096, 16384, 65536):
    noise = torch.empty((K, H), dtype=torch.float64, device=dev)
    noise_philox(3, 0, noise)
    cost = torch.as_tensor(np.random.default_rng(0).uniform(0, 3, K + 1), device=dev)
    us = torch.full((H,), -6.0, dtype=torch.float64, device=dev)
    part = torch.empty(H + 2, dtype=torch.float64, device=dev)
    for lam, tag in ((50.0, "all rows weighted"), (0.05, "few rows weighted")):
        t = queued_time(lambda s: plan.mppi_partial(cost, us, noise, 2.0, lam, partial=part,
                                                   stream=s))
        nbytes = (K + 1) * 8 + (K * H * 8 if lam > 1 else 0)
        print(json.dumps({"kernel": "mppi_partial_chunked_kernel", "rows": K + 1, "lambda": lam,
                          "note": tag, "us": round(t, 2),
                          "algorithmic_GB_s": round(nbytes / t * 1e-3, 1) if lam > 1 else None}))
    flag = torch.zeros(1, dtype=torch.int32, device=dev)

    def tail(s):
        plan.mppi_partial(cost, us, noise, 2.0, 50.0, partial=part, stream=s)
        mppi_combine(part.view(1, -1), 50.0, us2, flag, stream=s)

    us2 = us.clone()
    t = queued_time(tail)
    print(json.dumps({"kernel": "partial + combine (iteration tail)", "rows": K + 1, "us": round(t, 2)}))
    t = queued_time(lambda s: noise_philox(3, 0, noise, stream=s))
    print(json.dumps({"kernel": "noise_philox_kernel", "rows": K, "us": round(t, 2),
                      "algorithmic_GB_s": round(K * H * 8 / t * 1e-3, 1)}))
