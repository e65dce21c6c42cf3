"""Time one C4 candidate batch (K=4096+1, H=50, N=512 + ring) of the rollout kernel
under different launch shapes (VPM_SHAPE="nt,r,w0", VPM_MAXREG) -- a tuning tool;
results are shape-independent, only the time changes."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2509_16079_b200.device import DevicePlan  # noqa: E402

torch.cuda.set_device(0)
name = sys.argv[1] if len(sys.argv) > 1 else "scenario_C4.npz"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
shapes = sys.argv[3].split(";") if len(sys.argv) > 3 else ["default"]
with np.load(os.path.join("tests", "golden", name)) as z:
    sc = {k: z[k] for k in z.files}
flat = (sc["wake_pos"], sc["wake_gamma"], sc["wake_age"], int(sc["n_wake"]), int(sc["ring_a"]),
        int(sc["ring_b"]), sc["prev_pos"], sc["prev_gamma"], int(sc["n_prev"]), float(sc["prev_lev"]),
        sc["ema"])
plan = DevicePlan(sc["iparams"], sc["fparams"])
plan.set_fluid(flat)
dev = torch.device("cuda")
f64 = lambda a: torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64), device=dev)
noise = f64(np.random.default_rng(3).normal(0, 1, (K, 50)))
q = f64([10, 10, 1, 0, 0.2, 0.2, 0.2])
xp = f64([3.5, 0, np.pi / 4, 0, 0.5, -0.5, 0])
x0, us = f64(sc["x0"]), f64(sc["warm"])
ref = None
for shp in shapes:
    for key in ("VPM_SHAPE", "VPM_MAXREG"):
        os.environ.pop(key, None)
    if shp != "default":
        parts = shp.split("/")
        os.environ["VPM_SHAPE"] = parts[0]
        if len(parts) > 1:
            os.environ["VPM_MAXREG"] = parts[1]
    out = None
    for _ in range(2):
        out = plan.batch(x0, 50, ustar=us, noise=noise, sigma=2.0, rows=K + 1, q=q, x_perch=xp, out=out)
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        plan.batch(x0, 50, ustar=us, noise=noise, sigma=2.0, rows=K + 1, q=q, x_perch=xp, out=out)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    fin = out["finals"].cpu().numpy()
    same = None if ref is None else bool(np.array_equal(fin, ref))
    ref = fin if ref is None else ref
    print(json.dumps({"shape": shp, "ms": min(ts), "bitwise_equal_to_first": same}), flush=True)
