"""One replanning cycle on the GPU (API of perchsim/nmpc.py:40-164: ``ReplanRequest``,
``project_forward``, ``replan``, ``bootstrap_policy``).

``replan`` keeps every intermediate on the device: the closed-loop projection
(10 ``Engine.step`` calls under the current feedback policy) writes its final wake
straight into the plan's snapshot, the MPPI iterations, the nominal rollout, the
perturbed cloud and the regression + Riccati all fork from it.  The host only
synchronises at the reference's decision points -- projection failed, empty tail,
every candidate failed, nominal failed, fewer than 6 cloud survivors, Riccati
diverged -- and draws random numbers from the caller's generator in exactly the
reference's order (nothing is drawn on a path the reference would not reach).
"""

from __future__ import annotations

import dataclasses
from dataclasses import dataclass

import numpy as np

from . import mppi
from .config import ExperimentConfig
from .device import policy_fit
from .policy import NominalTrajectory, Policy, RankDeficientData, build_policy
from .rollout import Engine
from .vpm import FluidState


@dataclass
class ReplanRequest:
    x: np.ndarray
    fluid: FluidState
    policy: Policy
    t: float
    t_proj: int


def _dev(engine: Engine):
    import torch
    plan = mppi.engine_plan(engine)
    dev = torch.device("cuda", plan.device)
    return torch, plan, dev, (lambda a: torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64),
                                                        device=dev))


def _projection_time(t: float, t_proj: int, dt: float) -> float:
    for _ in range(t_proj):
        t += dt  # same accumulation as nmpc.py:102
    return t


def project_forward(policy: Policy, x, fluid: FluidState, t: float, t_proj: int, engine: Engine):
    """Advance the snapshot t_proj closed-loop steps under the policy (nmpc.py:88-103).
    Returns (x, fluid, t) or None on failure."""
    torch, plan, dev, f64 = _dev(engine)
    plan.set_fluid(fluid)
    nom = policy.nominal
    status, final = plan.project(f64(x), int(t_proj), f64(policy.gains), f64(nom.states),
                                 f64(nom.inputs), nom.t_start, float(t), write_snapshot=True)
    if int(status.item()) != 0:
        return None
    flat = plan.download_fluid()
    return final[0].cpu().numpy(), engine._rebuild(flat), _projection_time(t, t_proj, engine.cfg.dt)


def replan(req: ReplanRequest, cfg: ExperimentConfig, engine: Engine,
           rng: np.random.Generator) -> Policy | None:
    """Project, re-optimise, rebuild the policy (nmpc.py:106-134); None when rejected."""
    torch, plan, dev, f64 = _dev(engine)
    dt = engine.cfg.dt
    lim = engine.params.u_limit
    plan.set_fluid(req.fluid)
    old = req.policy.nominal
    # 1. closed-loop projection; its wake becomes the plan's snapshot on the device
    status, xdev = plan.project(f64(req.x), int(req.t_proj), f64(req.policy.gains),
                                f64(old.states), f64(old.inputs), old.t_start, float(req.t),
                                write_snapshot=True)
    if int(status.item()) != 0:
        return None
    t_new = _projection_time(float(req.t), int(req.t_proj), dt)
    k0 = int(round((t_new - old.t_start) / dt))
    tail = old.inputs[k0:]
    if len(tail) == 0:
        return None
    x0 = xdev[0]
    # 2. MPPI iterations (mppi.py:62-84) on the projected state and wake
    mc = cfg.mppi
    u = f64(np.clip(np.asarray(tail, dtype=float), -lim, lim))
    H, K, iters = u.shape[0], int(mc.batch), int(mc.iterations)
    if H and iters and K:
        scratch = {"cost": torch.empty(K + 1, dtype=torch.float64, device=dev),
                   "partial": torch.empty(H + 2, dtype=torch.float64, device=dev),
                   "flag": torch.zeros(1, dtype=torch.int32, device=dev)}
        q, xp = f64(mc.q_terminal), f64(mc.x_perch)
        for _ in range(iters):  # one draw per iteration, as mppi.py:42 (stops on failure)
            noise = f64(rng.normal(0.0, 1.0, (K, H)))
            plan.mppi_iteration(x0, u, noise, mc.input_stdev, K + 1, mc.temperature, q, xp, scratch)
            if int(scratch["flag"].item()) != 0:
                return None  # mppi.optimize raised ValueError
    # 3. nominal rollout of the new plan (nmpc.py:127)
    nomout = plan.batch(x0, H, controls=u.view(1, H), rows=1, record=True)
    if int(nomout["status"].item()) != 0:
        return None
    traj = nomout["trajs"][0]
    # 4. policy synthesis around it (policy.py:247-266): cloud, regression, Riccati
    sc = cfg.synthesis
    k = int(sc.n_samples)
    dx0 = f64(rng.normal(0.0, 1.0, (k, 7)))
    du = f64(rng.normal(0.0, 1.0, (k, H)))
    cstat, ctraj = plan.cloud(traj[0].contiguous(), dx0, f64(sc.state_stdev), u, du, sc.input_stdev)
    survivors = int((cstat == 0).sum().item())
    if survivors < 6:
        return None  # RankDeficientData
    cu = torch.clamp(u.view(1, H) + du * sc.input_stdev, -lim, lim)
    _, _, _, _, gains, flag = policy_fit(traj.contiguous(), u, ctraj, cu, cstat, dt, f64(sc.q_running),
                                         sc.r_running, f64(sc.q_final))
    if int(flag[0].item()) != 0:
        return None  # FloatingPointError
    nominal = NominalTrajectory(states=traj.cpu().numpy(), inputs=u.cpu().numpy(), dt=dt,
                                t_start=t_new)
    return Policy(gains=gains.cpu().numpy(), nominal=nominal,
                  q_final=np.asarray(sc.q_final, dtype=float))


def bootstrap_policy(cfg: ExperimentConfig, engine: Engine, rng: np.random.Generator) -> Policy:
    """Initial plan from rest (nmpc.py:137-164): annealed MPPI from a zero warm start
    (sigma x 1, 0.5, 0.25), nominal rollout, policy."""
    x0 = np.asarray(cfg.scenario.x0, dtype=float)
    fluid0 = FluidState.empty(cfg.vpm)
    u_star = np.zeros(cfg.mppi.horizon)
    total = cfg.scenario.bootstrap_iterations
    stage = max(1, total // 3)
    for scale, iters in ((1.0, stage), (0.5, stage), (0.25, total - 2 * stage)):
        if iters <= 0:
            continue
        stage_cfg = dataclasses.replace(cfg.mppi, input_stdev=cfg.mppi.input_stdev * scale)
        u_star = mppi.optimize(x0, fluid0, u_star, stage_cfg, engine, rng, iterations=iters)
    rc, traj, _ = engine.rollout(x0, u_star, fluid0, record=True)
    if rc != 0:
        raise RuntimeError("bootstrap nominal rollout failed")
    nominal = NominalTrajectory(states=traj, inputs=u_star, dt=cfg.vpm.dt, t_start=0.0)
    return build_policy(nominal, fluid0, cfg.synthesis, engine, rng)


__all__ = ["ReplanRequest", "project_forward", "replan", "bootstrap_policy", "RankDeficientData"]
