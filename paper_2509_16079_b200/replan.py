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
from .device import noise_philox, policy_fit
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
    with plan.lock:
        return _project_locked(plan, f64, policy, x, fluid, t, t_proj, engine)


def _project_locked(plan, f64, policy, x, fluid, t, t_proj, engine):
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
    """Project, re-optimise, rebuild the policy (nmpc.py:106-134); None when rejected.

    The whole cycle is queued on one stream with a single host synchronisation at
    the end: projection -> MPPI iterations -> one launch of the nominal rollout
    (row 0, zero perturbation: bitwise the reference's ``rollout(x_proj, u*)``)
    together with the 64-rollout cloud (rows 1..64) -> regression + Riccati.  The
    random numbers of the success path are drawn in the reference's order
    (iteration noises, then the cloud's dx0 and du), each while the device runs
    the previous launch.
    The reference stops drawing at its first failure (nmpc.py:118-134); when the
    cycle turns out to have failed at such a point, the generator is rewound and
    exactly the draws the reference made before failing are replayed, so the
    caller's generator ends in the reference's state either way.
    With ``rng = mppi.DeviceNoise(seed)`` (performance mode) every draw -- the MPPI
    noise and the cloud's dx0 / du -- is made on the device instead and no host
    random numbers are generated.
    """
    torch, plan, dev, _ = _dev(engine)
    with plan.lock:
        return _replan_locked(torch, plan, dev, req, cfg, engine, rng)


def _replan_locked(torch, plan, dev, req, cfg, engine, rng):
    dt = engine.cfg.dt
    lim = engine.params.u_limit
    old = req.policy.nominal
    t_new = _projection_time(float(req.t), int(req.t_proj), dt)
    k0 = int(round((t_new - old.t_start) / dt))
    tail = old.inputs[k0:]
    if len(tail) == 0:
        return None  # nothing to re-plan; the reference draws nothing on this path either
    plan.set_fluid(req.fluid)
    mc, sc = cfg.mppi, cfg.synthesis
    H, K, iters, k = len(tail), int(mc.batch), int(mc.iterations), int(sc.n_samples)
    run_mppi = bool(H and iters and K)
    # Every small input goes up in ONE non-blocking copy from the pinned staging
    # buffer: a torch.as_tensor of a pageable numpy array would synchronise the
    # stream and stall the host behind the launches already queued.
    gains = np.asarray(req.policy.gains, dtype=float)
    states = np.asarray(old.states, dtype=float)
    inputs = np.asarray(old.inputs, dtype=float)
    parts = [np.clip(np.asarray(tail, dtype=float), -lim, lim), np.asarray(req.x, dtype=float), gains,
             states, inputs, np.asarray(mc.q_terminal, dtype=float), np.asarray(mc.x_perch, dtype=float),
             np.asarray(sc.state_stdev, dtype=float), np.asarray(sc.q_running, dtype=float),
             np.asarray(sc.q_final, dtype=float)]
    offs = np.cumsum([0] + [a.size for a in parts])
    nh = int(offs[-1])
    n_it = K * H if run_mppi else 0
    n_cloud = (k + 1) * 7 + (k + 1) * H
    host = plan.staging(nh + iters * n_it + n_cloud)
    hv = host.numpy()
    for a, o in zip(parts, offs[:-1]):
        hv[o:o + a.size] = a.ravel()
    head = host[:nh].to(dev, non_blocking=True)
    seg = [head[offs[i]:offs[i + 1]] for i in range(len(parts))]
    u = seg[0]  # u* (updated in place by the MPPI iterations)
    d_x, d_gains, d_states, d_inputs = seg[1], seg[2].view(gains.shape), seg[3].view(states.shape), seg[4]
    q, xp, d_sx, d_qr, d_qf = seg[5], seg[6], seg[7], seg[8], seg[9]
    # 1. closed-loop projection; its wake becomes the plan's snapshot on the device
    pstat, xdev = plan.project(d_x, int(req.t_proj), d_gains, d_states, d_inputs, old.t_start,
                               float(req.t), write_snapshot=True)
    x0 = xdev[0]
    # 2./3. the success path's draws and the MPPI iterations (mppi.py:62-84),
    # pipelined: each iteration's noise is drawn on the host and copied while the
    # device runs the previous launch; one failure flag per iteration
    # performance mode (mppi.DeviceNoise): every draw on the device, no host RNG
    devnoise = isinstance(rng, mppi.DeviceNoise)
    saved = None if devnoise else rng.bit_generator.state
    flags = torch.zeros(max(iters, 1), dtype=torch.int32, device=dev)
    if run_mppi:
        scratch = {"cost": torch.empty(K + 1, dtype=torch.float64, device=dev),
                   "partial": torch.empty(H + 2, dtype=torch.float64, device=dev)}
        d_buf = torch.empty((K, H), dtype=torch.float64, device=dev) if devnoise else None
        for i in range(iters):
            if devnoise:
                d_noise = noise_philox(rng.seed, rng.iteration + i, d_buf)
            else:
                lo = nh + i * n_it
                hv[lo:lo + n_it] = rng.normal(0.0, 1.0, (K, H)).ravel()
                d_noise = host[lo:lo + n_it].to(dev, non_blocking=True).view(K, H)
            scratch["flag"] = flags[i:i + 1]
            plan.mppi_iteration(x0, u, d_noise, mc.input_stdev, K + 1, mc.temperature, q, xp, scratch)
    if devnoise:
        dcl = torch.zeros(n_cloud, dtype=torch.float64, device=dev)  # row 0: the nominal
        d_cx = dcl[:(k + 1) * 7].view(k + 1, 7)
        d_cu = dcl[(k + 1) * 7:].view(k + 1, H)
        if k > 0:
            noise_philox(rng.seed, rng.iteration + iters, d_cx[1:])
            noise_philox(rng.seed, rng.iteration + iters + 1, d_cu[1:])
        rng.iteration += iters + 2
    else:
        lo = nh + iters * n_it
        dx0 = rng.normal(0.0, 1.0, (k, 7))
        du = rng.normal(0.0, 1.0, (k, H))
        cx = hv[lo:lo + (k + 1) * 7].reshape(k + 1, 7)
        cu = hv[lo + (k + 1) * 7:lo + n_cloud].reshape(k + 1, H)
        cx[0], cx[1:] = 0.0, dx0  # row 0: the nominal, unperturbed
        cu[0], cu[1:] = 0.0, du
        dcl = host[lo:lo + n_cloud].to(dev, non_blocking=True)
        d_cx = dcl[:(k + 1) * 7].view(k + 1, 7)
        d_cu = dcl[(k + 1) * 7:].view(k + 1, H)
    # 4. nominal (row 0) + perturbed cloud (rows 1..k) in one launch (policy.py:66-91)
    cstat, ctraj = plan.cloud(x0, d_cx, d_sx, u, d_cu, sc.input_stdev)
    traj = ctraj[0]
    cu_dev = torch.clamp(u.view(1, H) + d_cu[1:] * sc.input_stdev, -lim, lim)
    # 5. regression + Riccati around the nominal (policy.py:247-266)
    _, _, _, _, d_gain, fflag = policy_fit(traj, u, ctraj[1:], cu_dev, cstat[1:], dt, d_qr, sc.r_running,
                                           d_qf)
    # 6. the one synchronisation: every decision the reference makes, in its order
    ints = torch.cat([pstat.view(1), flags.to(torch.int64), cstat, fflag[:1].to(torch.int64)]).cpu().numpy()
    if devnoise:  # no generator to leave in the reference's state
        st = ints[1 + max(iters, 1):1 + max(iters, 1) + k + 1]
        if ints[0] != 0 or (run_mppi and np.any(ints[1:1 + iters] != 0)) or st[0] != 0:
            return None
        if int((st[1:] == 0).sum()) < 6 or ints[-1] != 0:
            return None
        nominal = NominalTrajectory(states=traj.cpu().numpy(), inputs=u.cpu().numpy(), dt=dt, t_start=t_new)
        return Policy(gains=d_gain.cpu().numpy(), nominal=nominal, q_final=np.asarray(sc.q_final, dtype=float))
    if ints[0] != 0:
        rng.bit_generator.state = saved  # projection failed before any draw
        return None
    for i in range(iters if run_mppi else 0):
        if ints[1 + i] != 0:  # mppi.optimize raised ValueError after drawing i + 1 noises
            rng.bit_generator.state = saved
            rng.normal(0.0, 1.0, (i + 1, K, H))
            return None
    st = ints[1 + max(iters, 1):1 + max(iters, 1) + k + 1]
    if st[0] != 0:  # nominal rollout failed: the reference drew the MPPI noise only
        rng.bit_generator.state = saved
        if run_mppi:
            rng.normal(0.0, 1.0, (iters, K, H))
        return None
    if int((st[1:] == 0).sum()) < 6 or ints[-1] != 0:
        return None  # RankDeficientData / FloatingPointError after all draws
    nominal = NominalTrajectory(states=traj.cpu().numpy(), inputs=u.cpu().numpy(), dt=dt, t_start=t_new)
    return Policy(gains=d_gain.cpu().numpy(), nominal=nominal, q_final=np.asarray(sc.q_final, dtype=float))


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
