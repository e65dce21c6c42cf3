"""Single-instance stepping latency split (tuning tool): host wall time per resident
DeviceWake step (launch + sync) next to the step's device time (CUDA events around 200
queued steps without syncs), and Engine.step with host buffers."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2509_16079_b200 import config, rollout, vpm  # noqa: E402
from paper_2509_16079_b200.plant import DeviceWake  # noqa: E402

torch.cuda.set_device(0)
for cap in (60, 512):
    cfg = config.ExperimentConfig()
    cfg.vpm.particle_cap = cap
    eng = rollout.Engine(cfg.vpm, cfg.glider)
    fl = vpm.FluidState.empty(cfg.vpm)
    x0 = np.array([0.0, 0.0, 0.3, 0.0, 7.0, 0.0, 0.0])
    dw = DeviceWake(eng, fl)
    for _ in range(min(cap - 4, 200)):  # grow the wake
        dw.step_async(x0, -6.0, True)
        dw.sync()
    n = 200
    t0 = time.perf_counter()
    for _ in range(n):
        dw.step_async(x0, -6.0, True)
        dw.sync()
    wall = 1e6 * (time.perf_counter() - t0) / n
    t0 = time.perf_counter()
    for _ in range(n):
        dw.step_async(x0, -6.0, True)
    host = 1e6 * (time.perf_counter() - t0) / n
    dw.sync()
    s = dw.stream
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        torch.cuda._sleep(50_000_000)
        e0.record(s)
    for _ in range(n):
        dw.step_async(x0, -6.0, True)
    with torch.cuda.stream(s):
        e1.record(s)
    dw.sync()
    dev = 1e3 * e0.elapsed_time(e1) / n
    t0 = time.perf_counter()
    for _ in range(n):
        eng.step(x0, -6.0, fl)
    es = 1e6 * (time.perf_counter() - t0) / n
    print(f"cap {cap}: resident step {wall:.1f} us wall (host enqueue {host:.1f} us, device per queued "
          f"step {dev:.1f} us); Engine.step with host buffers {es:.1f} us")
