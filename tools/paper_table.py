"""The paper's runtime table (80-step batched rollouts, <= 60
particles, batch 1/128/256/512/1024) on B200, next to the reference's compiled CPU
core (oracle/_ref, all host threads) on the same inputs.

Inputs: x0 = [0,0,0.3,0,7,0,0]; controls
clip(-15 + N(0, 2^2)); empty initial wake, cap 60, H = 80.  GPU time: CUDA events
around the device batch (inputs resident); e2e: the reference-facing
Engine.batch call with host buffers.  Prints one JSON line.
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2509_16079_b200 import config, rollout, vpm  # noqa: E402
from paper_2509_16079_b200.device import DevicePlan  # noqa: E402

PAPER_RTX5080_MS = {1: 8.0, 128: 10.3, 256: 12.2, 512: 16.3, 1024: 27.2}


def main():
    torch.cuda.set_device(0)
    cfg = config.ExperimentConfig()  # particle_cap = 60
    eng = rollout.Engine(cfg.vpm, cfg.glider)
    fl = vpm.FluidState.empty(cfg.vpm)
    x0 = np.array([0.0, 0.0, 0.3, 0.0, 7.0, 0.0, 0.0])
    plan = DevicePlan(eng.iparams, eng.fparams)
    plan.set_fluid(fl)
    dev = torch.device("cuda")
    ref = None
    try:
        from oracle import refcore
        ref = refcore.load()
    except Exception:
        ref = None
    rows = {}
    for B in (1, 128, 256, 512, 1024):
        u = np.clip(-15.0 + 2.0 * np.random.default_rng(B).normal(0.0, 1.0, (B, 80)), -15, 15)
        ud = torch.as_tensor(u, device=dev)
        xd = torch.as_tensor(x0, device=dev)
        out = plan.batch(xd, 80, controls=ud, rows=B)
        torch.cuda.synchronize()
        best = float("inf")
        for _ in range(5):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            plan.batch(xd, 80, controls=ud, rows=B, out=out)
            b.record()
            torch.cuda.synchronize()
            best = min(best, a.elapsed_time(b))
        eng.batch(rollout.RolloutRequest(x0=x0, fluid=fl, controls=u))
        t0 = time.perf_counter()
        for _ in range(5):
            eng.batch(rollout.RolloutRequest(x0=x0, fluid=fl, controls=u))
        e2e = 1e3 * (time.perf_counter() - t0) / 5
        row = {"gpu_ms": best, "e2e_ms": e2e, "paper_rtx5080_ms": PAPER_RTX5080_MS[B]}
        if ref is not None:
            t0 = time.perf_counter()
            ref.batch_rollout(x0, np.ascontiguousarray(u), *fl.flat(), eng.iparams, eng.fparams, False,
                              os.cpu_count() or 1)
            row["cpu_reference_ms"] = 1e3 * (time.perf_counter() - t0)
        rows[str(B)] = row
    print(json.dumps({"table": "80-step batched rollouts, cap 60 (PAPER.md:404-418)",
                      "cpu_cores": os.cpu_count(), "by_batch": rows}))


if __name__ == "__main__":
    main()
