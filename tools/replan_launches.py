"""Drive replanning cycles at the paper's operating point (bench.py extras: 10-step
projection, 3 MPPI iterations K=256 over the 67-step tail, nominal, policy; cap 60)
with device noise, for a launch-list capture (tuning tool):
  ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/replan_launches.py
Without ncu it prints the end-to-end time per cycle."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2509_16079_b200 import config, mppi, rollout, vpm  # noqa: E402
from paper_2509_16079_b200 import replan as rp  # noqa: E402
from paper_2509_16079_b200.policy import NominalTrajectory, Policy  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
with np.load(os.path.join(ROOT, "tests", "golden", "nmpc_replan.npz")) as z:
    gr = {k: z[k] for k in z.files}
cfg = config.ExperimentConfig()
eng = rollout.Engine.from_config(cfg)
pol = Policy(gains=gr["boot_gains"], nominal=NominalTrajectory(gr["boot_states"], gr["boot_inputs"], 0.01))
req = rp.ReplanRequest(x=np.asarray(cfg.scenario.x0, float), fluid=vpm.FluidState.empty(cfg.vpm), policy=pol,
                       t=0.0, t_proj=10)
n = int(os.environ.get("REPLAN_CYCLES", "4"))
for i in range(n):
    t0 = time.perf_counter()
    rp.replan(req, cfg, eng, mppi.DeviceNoise(i))
    print(f"cycle {i}: {1e3 * (time.perf_counter() - t0):.3f} ms e2e", flush=True)
