"""Per-phase cycle breakdown of rollout 0 (needs a library built with
-DVPM_PHASE_TIMING, selected with VPM_LIB=...).  Usage:
  python tools/phase_timing.py scenario_C2.npz 256"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2509_16079_b200 import _lib  # noqa: E402
from paper_2509_16079_b200.device import DevicePlan  # noqa: E402

NAMES = ["P1 split", "B1 wait", "D geometry", "sweep+A", "B2 wait", "S2 split", "B3 wait", "E (warp0)", "B4 wait", "D loads", "D integrate", "D record"]
torch.cuda.set_device(0)
name = sys.argv[1] if len(sys.argv) > 1 else "scenario_C2.npz"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 256
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
L = _lib.lib()
fn = L.vpm_debug_phase_cycles
fn.restype = C.c_int
fn.argtypes = [C.c_void_p, C.c_int]
buf = np.zeros((2, 12), dtype=np.uint64)
out = plan.batch(f64(sc["x0"]), 50, ustar=f64(sc["warm"]), noise=noise, sigma=2.0, rows=K + 1)
torch.cuda.synchronize()
assert fn(buf.ctypes.data, 1) == 24, "library not built with -DVPM_PHASE_TIMING"
plan.batch(f64(sc["x0"]), 50, ustar=f64(sc["warm"]), noise=noise, sigma=2.0, rows=K + 1, out=out)
torch.cuda.synchronize()
fn(buf.ctypes.data, 0)
tot = buf[0, :12].sum()
print(name, "K", K, "rollout-0 cycles per step (50 steps): total", tot / 50)
for i, nm in enumerate(NAMES[:12]):
    print(f"  {nm:10s} warp0 {buf[0, i] / 50:9.0f}   warp1 {buf[1, i] / 50:9.0f}")
