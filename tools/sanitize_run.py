"""Small invocations of every kernel, for compute-sanitizer (memcheck / racecheck /
synccheck):  compute-sanitizer --tool racecheck python tools/sanitize_run.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2509_16079_b200 import mppi, policy, replan, rollout, vpm  # noqa: E402
from paper_2509_16079_b200.config import ExperimentConfig  # noqa: E402
from paper_2509_16079_b200.device import DevicePlan  # noqa: E402

torch.cuda.set_device(0)
dev = torch.device("cuda")
f64 = lambda a: torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64), device=dev)
for name, K, H in (("scenario_C4.npz", 3, 3), ("scenario_C3.npz", 3, 4), ("scenario_C2.npz", 8, 6)):
    with np.load(os.path.join("tests", "golden", name)) as z:
        sc = {k: z[k] for k in z.files}
    flat = (sc["wake_pos"], sc["wake_gamma"], sc["wake_age"], int(sc["n_wake"]), int(sc["ring_a"]),
            int(sc["ring_b"]), sc["prev_pos"], sc["prev_gamma"], int(sc["n_prev"]), float(sc["prev_lev"]),
            sc["ema"])
    plan = DevicePlan(sc["iparams"], sc["fparams"])
    plan.set_fluid(flat)
    noise = f64(np.random.default_rng(3).normal(0, 1, (K, H)))
    out = plan.batch(f64(sc["x0"]), H, ustar=f64(sc["warm"][:H]), noise=noise, sigma=2.0, rows=K + 1,
                     q=f64([10, 10, 1, 0, .2, .2, .2]), x_perch=f64([3.5, 0, .785, 0, .5, -.5, 0]),
                     record=True, diagnostics=True)
    torch.cuda.synchronize()
    print(name, out["status"].cpu().numpy())
# the symmetric sweep on odd / even tile counts with partial tiles (caps 640, 1000) and
# an overfull snapshot (direct fallback for the first step)
from paper_2509_16079_b200 import config  # noqa: E402
for cap, n0 in ((640, 600), (1000, 900), (512, 516)):
    rng = np.random.default_rng(cap)
    v = config.VpmConfig(particle_cap=cap)
    ip, fp = config.pack_params(v, config.GliderParams())
    p5 = DevicePlan(ip, fp)
    wp = rng.normal(0.0, 0.5, (n0, 2)) - np.array([3.0, 0.0])
    p5.set_fluid((wp, rng.normal(0.0, 0.02, n0), rng.integers(0, 300, n0), n0, -1, -1, np.zeros((10, 2)),
                  np.zeros(10), 0, 0.0, np.zeros(10)))
    ctrl = f64(np.clip(rng.normal(-6.0, 3.0, (2, 3)), -15, 15))
    out = p5.batch(f64([0.0, 0.0, 0.3, 0.0, 7.0, 0.0, 0.0]), 3, controls=ctrl, rows=2, diagnostics=True)
    torch.cuda.synchronize()
    print("cap", cap, out["status"].cpu().numpy())
cfg = ExperimentConfig()
eng = rollout.Engine.from_config(cfg)
fl = vpm.FluidState.empty(cfg.vpm)
x = np.array([0.0, 0.0, 0.3, 0.0, 7.0, 0.0, 0.0])
for _ in range(4):
    ok, x, fl, _ = eng.step(x, -6.0, fl)
u = mppi.optimize(x, fl, np.full(12, -6.0), cfg.mppi, eng, np.random.default_rng(0), iterations=1)
rc, traj, _ = eng.rollout(x, u, fl, record=True)
nom = policy.NominalTrajectory(traj, u, cfg.vpm.dt)
pol = policy.build_policy(nom, fl, cfg.synthesis, eng, np.random.default_rng(1))
new = replan.replan(replan.ReplanRequest(x=x, fluid=fl, policy=pol, t=0.0, t_proj=3), cfg, eng,
                    np.random.default_rng(2))
print("replan", new is not None)
print("induced", vpm.induced_velocity_at([[0.1, 0.2]], fl.wake_pos[:fl.n_wake], fl.wake_gamma[:fl.n_wake], r_core=0.02))
# device-noise optimiser (noise kernel + MPPI partial / combine)
u2 = mppi.optimize(x, fl, np.full(12, -6.0), cfg.mppi, eng, mppi.DeviceNoise(4), iterations=2)
torch.cuda.synchronize()
print("device noise ok", np.isfinite(u2).all())
