"""One C2 MPPI candidate batch (K=256+1, H=50, cap 60, empty fluid): the
latency-bound configuration, for profiling the per-step serial chain."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2509_16079_b200.device import DevicePlan  # noqa: E402

torch.cuda.set_device(0)
with np.load(os.path.join("tests", "golden", "scenario_C2.npz")) as z:
    sc = {k: z[k] for k in z.files}
plan = DevicePlan(sc["iparams"], sc["fparams"])
plan.set_fluid((sc["wake_pos"], sc["wake_gamma"], sc["wake_age"], 0, -1, -1, sc["prev_pos"],
                sc["prev_gamma"], 0, 0.0, sc["ema"]))
dev = torch.device("cuda")
f64 = lambda a: torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64), device=dev)
noise = f64(np.random.default_rng(3).normal(0, 1, (256, 50)))
q, xp = f64([10, 10, 1, 0, 0.2, 0.2, 0.2]), f64([3.5, 0, np.pi / 4, 0, 0.5, -0.5, 0])
out = None
for _ in range(4):
    out = plan.batch(f64(sc["x0"]), 50, ustar=f64(sc["warm"]), noise=noise, sigma=2.0, rows=257, q=q,
                     x_perch=xp, out=out)
torch.cuda.synchronize()
print("ok", int((out["status"] == 0).sum().item()))
