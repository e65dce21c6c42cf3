"""Timing suite for kernel-variant A/B runs (select the library with VPM_LIB=...):
one 50-step batch launch at 4097 / 2049 / 1025 / 513 rows on the C4 snapshot, the C2
batch (257 rows, cap 60) and one full replan cycle (nmpc.replan) end to end.
Prints one JSON line; device times are the min of 5 CUDA-event timed launches."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2509_16079_b200.device import DevicePlan  # noqa: E402

torch.cuda.set_device(0)
dev = torch.device("cuda")
f64 = lambda a: torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64), device=dev)
res = {"lib": os.environ.get("VPM_LIB", "default")}


def flat_of(sc):
    return (sc["wake_pos"], sc["wake_gamma"], sc["wake_age"], int(sc["n_wake"]), int(sc["ring_a"]),
            int(sc["ring_b"]), sc["prev_pos"], sc["prev_gamma"], int(sc["n_prev"]), float(sc["prev_lev"]),
            sc["ema"])


def time_batch(name, K):
    with np.load(os.path.join("tests", "golden", name)) as z:
        sc = {k: z[k] for k in z.files}
    plan = DevicePlan(sc["iparams"], sc["fparams"])
    plan.set_fluid(flat_of(sc))
    noise = f64(np.random.default_rng(3).normal(0, 1, (K, 50)))
    q = f64([10, 10, 1, 0, 0.2, 0.2, 0.2])
    xp = f64([3.5, 0, np.pi / 4, 0, 0.5, -0.5, 0])
    x0, us = f64(sc["x0"]), f64(sc["warm"])
    out = None
    for _ in range(2):
        out = plan.batch(x0, 50, ustar=us, noise=noise, sigma=2.0, rows=K + 1, q=q, x_perch=xp, out=out)
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        plan.batch(x0, 50, ustar=us, noise=noise, sigma=2.0, rows=K + 1, q=q, x_perch=xp, out=out)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return min(ts)


for K in (4096, 2048, 1024, 512):
    res[f"c4_rows{K + 1}_ms"] = time_batch("scenario_C4.npz", K)
res["c2_rows257_ms"] = time_batch("scenario_C2.npz", 256)

from paper_2509_16079_b200 import config, replan as rp, rollout, vpm  # noqa: E402
from paper_2509_16079_b200.policy import NominalTrajectory, Policy  # noqa: E402

with np.load(os.path.join("tests", "golden", "nmpc_replan.npz")) as z:
    gr = {k: z[k] for k in z.files}
cfg = config.ExperimentConfig()
eng = rollout.Engine.from_config(cfg)
pol = Policy(gains=gr["boot_gains"], nominal=NominalTrajectory(gr["boot_states"], gr["boot_inputs"], 0.01))
req = rp.ReplanRequest(x=np.asarray(cfg.scenario.x0, float), fluid=vpm.FluidState.empty(cfg.vpm),
                       policy=pol, t=0.0, t_proj=10)
rp.replan(req, cfg, eng, np.random.default_rng(1))
best = 1e9
for i in range(5):
    t0 = time.perf_counter()
    rp.replan(req, cfg, eng, np.random.default_rng(1 + i))
    best = min(best, time.perf_counter() - t0)
res["replan_cycle_ms"] = best * 1e3
print(json.dumps(res), flush=True)
