"""Run nmpc.replan (the paper's operating point, cap 60, K=256) a few times -- the
target of the replan-cycle ncu launch list / policy_kernel capture."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2509_16079_b200 import config, replan as rp, rollout, vpm  # noqa: E402
from paper_2509_16079_b200.policy import NominalTrajectory, Policy  # noqa: E402

torch.cuda.set_device(0)
with np.load(os.path.join("tests", "golden", "nmpc_replan.npz")) as z:
    gr = {k: z[k] for k in z.files}
cfg = config.ExperimentConfig()
eng = rollout.Engine.from_config(cfg)
pol = Policy(gains=gr["boot_gains"], nominal=NominalTrajectory(gr["boot_states"], gr["boot_inputs"], 0.01))
req = rp.ReplanRequest(x=np.asarray(cfg.scenario.x0, float), fluid=vpm.FluidState.empty(cfg.vpm),
                       policy=pol, t=0.0, t_proj=10)
for i in range(int(sys.argv[1]) if len(sys.argv) > 1 else 3):
    out = rp.replan(req, cfg, eng, np.random.default_rng(1 + i))
    assert out is not None
torch.cuda.synchronize()
print("ok")
