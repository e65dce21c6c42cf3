"""C5 Biot-Savart stress (K=16384 rollouts x H=5, attached flow, random wake of N
particles) under different launch shapes: VPM_SHAPE="nt,r" / VPM_MAXREG overrides.
usage: python tools/c5_shapes.py N "default;64,3/48;..."  (tuning tool)"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2509_16079_b200 import config  # noqa: E402
from paper_2509_16079_b200.device import DevicePlan  # noqa: E402

torch.cuda.set_device(0)
dev = torch.device("cuda")
N = int(sys.argv[1])
shapes = sys.argv[2].split(";") if len(sys.argv) > 2 else ["default"]
K5, H5 = int(os.environ.get("C5_K", "16384")), int(os.environ.get("C5_H", "5"))
rng = np.random.default_rng(11)
v = config.VpmConfig(particle_cap=N)
ip, fp = config.pack_params(v, config.GliderParams())
plan = DevicePlan(ip, fp)
wp = rng.normal(0.0, 0.5, (N, 2))
wp[:, 0] -= 3.0
plan.set_fluid((wp, rng.normal(0.0, 0.05, N), np.zeros(N, np.int64), N, -1, -1, np.zeros((10, 2)),
                np.zeros(10), 0, 0.0, np.zeros(10)))
x5 = torch.tensor([0.0, 0.0, 0.0, 0.0, 7.0, 0.0, 0.0], dtype=torch.float64, device=dev)
ctrl = torch.zeros(K5, H5, dtype=torch.float64, device=dev)
o5 = {"status": torch.empty(K5, dtype=torch.int64, device=dev),
      "finals": torch.empty(K5, 7, dtype=torch.float64, device=dev),
      "interactions": torch.zeros(K5, dtype=torch.int64, device=dev)}
ref = None
for shp in shapes:
    for key in ("VPM_SHAPE", "VPM_MAXREG"):
        os.environ.pop(key, None)
    if shp != "default":
        parts = shp.split("/")
        os.environ["VPM_SHAPE"] = parts[0]
        if len(parts) > 1:
            os.environ["VPM_MAXREG"] = parts[1]
    plan.batch(x5, H5, controls=ctrl, rows=K5, out=o5)
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        plan.batch(x5, H5, controls=ctrl, rows=K5, out=o5)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    inter = float(o5["interactions"].sum().item())
    fin = o5["finals"].cpu().numpy()
    same = None if ref is None else bool(np.array_equal(fin, ref))
    ref = fin if ref is None else ref
    ms = min(ts)
    print(json.dumps({"N": N, "shape": shp, "ms": ms, "frac_fp32": 12 * inter / (ms * 1e-3) / 74.45e12,
                      "bitwise_equal_to_first": same}), flush=True)
