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
from .device import noise_philox, noise_philox_dev, policy_fit
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
           rng: np.random.Generator, graph: bool = True) -> Policy | None:
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
    random numbers are generated; the whole cycle is then captured once per shape
    as a CUDA graph and replayed (``graph=False``: queued launch by launch; both
    give the same bits).
    """
    torch, plan, dev, _ = _dev(engine)
    with plan.lock:
        if graph and isinstance(rng, mppi.DeviceNoise):
            return _replan_graphed(torch, plan, dev, req, cfg, engine, rng)
        return _replan_locked(torch, plan, dev, req, cfg, engine, rng)


class _ReplanGraph:
    """A device-noise replan cycle captured as one CUDA graph for a fixed shape
    (old-policy length, tail length H, K, iterations, cloud size, projection steps):
    projection (times read on the device) -> iterations x (Philox noise with
    seed / iteration read on the device + rollouts + partial + combine) -> nominal +
    cloud -> clamp -> regression + Riccati -> the decision flags, nominal, u* and
    gains copied to pinned host buffers.  Every per-call input -- the fluid snapshot
    (the plan's pinned mirror), the small inputs and the Philox seed / iteration --
    is copied up inside the graph from pinned memory at fixed addresses, so a
    replay needs no argument updates."""

    def __init__(self, torch, plan, dev, cfg, engine, hold: int, H: int, t_proj: int):
        self.torch, self.plan, self.dev = torch, plan, dev
        mc, sc = cfg.mppi, cfg.synthesis
        self.K, self.iters, self.k, self.H, self.hold, self.t_proj = (int(mc.batch), int(mc.iterations),
                                                                      int(sc.n_samples), H, hold, t_proj)
        self.sizes = [H, 7, hold * 7, (hold + 1) * 7, hold, 7, 7, 7, 7, 7, 2]
        self.offs = np.cumsum([0] + self.sizes)
        f64, i64 = torch.float64, torch.int64
        n_ints = 1 + max(self.iters, 1) + self.k + 1 + 1
        self.h_head = torch.zeros(int(self.offs[-1]), dtype=f64, pin_memory=True)
        self.h_si = torch.zeros(2, dtype=i64, pin_memory=True)
        self.h_ints = torch.zeros(n_ints, dtype=i64, pin_memory=True)
        self.h_traj = torch.zeros((H + 1) * 7, dtype=f64, pin_memory=True)
        self.h_u = torch.zeros(H, dtype=f64, pin_memory=True)
        self.h_gain = torch.zeros(H * 7, dtype=f64, pin_memory=True)
        self.d_head = torch.zeros(int(self.offs[-1]), dtype=f64, device=dev)
        self.d_si = torch.zeros(2, dtype=i64, device=dev)
        self.consts = (float(mc.input_stdev), float(mc.temperature), float(sc.input_stdev), float(sc.r_running),
                       float(engine.cfg.dt), float(engine.params.u_limit))
        stream = torch.cuda.Stream(dev)
        stream.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(stream):  # eager warm-up: scratch growth, kernel attributes
            self._body()
        stream.synchronize()
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph, stream=stream, capture_error_mode="thread_local"):
            self._body()
        stream.synchronize()

    def _body(self):
        torch, plan = self.torch, self.plan
        H, K, iters, k, hold = self.H, self.K, self.iters, self.k, self.hold
        sig, lam, sig_u, r_run, dt, lim = self.consts
        plan.upload_fluid()  # the snapshot staged in the plan's pinned mirror
        self.d_head.copy_(self.h_head, non_blocking=True)
        self.d_si.copy_(self.h_si, non_blocking=True)
        seg = [self.d_head[self.offs[i]:self.offs[i + 1]] for i in range(len(self.sizes))]
        u, d_x = seg[0], seg[1]
        d_gains, d_states, d_inputs = seg[2].view(hold, 7), seg[3].view(hold + 1, 7), seg[4]
        q, xp, d_sx, d_qr, d_qf, d_times = seg[5], seg[6], seg[7], seg[8], seg[9], seg[10]
        pstat, xdev = plan.project_dev(d_x, self.t_proj, d_gains, d_states, d_inputs, d_times)
        x0 = xdev[0]
        flags = torch.zeros(max(iters, 1), dtype=torch.int32, device=self.dev)
        if H and iters and K:
            scratch = {"cost": torch.empty(K + 1, dtype=torch.float64, device=self.dev),
                       "partial": torch.empty(H + 2, dtype=torch.float64, device=self.dev)}
            d_buf = torch.empty((K, H), dtype=torch.float64, device=self.dev)
            for i in range(iters):
                noise_philox_dev(self.d_si, i, d_buf)
                scratch["flag"] = flags[i:i + 1]
                plan.mppi_iteration(x0, u, d_buf, sig, K + 1, lam, q, xp, scratch)
        dcl = torch.zeros((k + 1) * 7 + (k + 1) * H, dtype=torch.float64, device=self.dev)
        d_cx = dcl[:(k + 1) * 7].view(k + 1, 7)
        d_cu = dcl[(k + 1) * 7:].view(k + 1, H)
        if k > 0:
            noise_philox_dev(self.d_si, iters, d_cx[1:])
            noise_philox_dev(self.d_si, iters + 1, d_cu[1:])
        cstat, ctraj = plan.cloud(x0, d_cx, d_sx, u, d_cu, sig_u)
        traj = ctraj[0]
        cu_dev = torch.clamp(u.view(1, H) + d_cu[1:] * sig_u, -lim, lim)
        _, _, _, _, d_gain, fflag = policy_fit(traj, u, ctraj[1:], cu_dev, cstat[1:], dt, d_qr, r_run, d_qf)
        ints = torch.cat([pstat.view(1), flags.to(torch.int64), cstat, fflag[:1].to(torch.int64)])
        self.h_ints.copy_(ints, non_blocking=True)
        self.h_traj.copy_(traj.reshape(-1), non_blocking=True)
        self.h_u.copy_(u, non_blocking=True)
        self.h_gain.copy_(d_gain.reshape(-1), non_blocking=True)

    def run(self, parts, seed: int, iteration: int):
        hv = self.h_head.numpy()
        for a, o in zip(parts, self.offs[:-1]):
            hv[o:o + a.size] = a.ravel()
        self.h_si.numpy()[:] = (np.int64(np.uint64(seed & (2**64 - 1)).view(np.int64)), iteration)
        self.graph.replay()
        self.torch.cuda.current_stream(self.dev).synchronize()
        return (self.h_ints.numpy().copy(), self.h_traj.numpy().reshape(self.H + 1, 7).copy(),
                self.h_u.numpy().copy(), self.h_gain.numpy().reshape(self.H, 7).copy())


def _replan_graphed(torch, plan, dev, req, cfg, engine, rng):
    dt = engine.cfg.dt
    lim = engine.params.u_limit
    old = req.policy.nominal
    t_new = _projection_time(float(req.t), int(req.t_proj), dt)
    k0 = int(round((t_new - old.t_start) / dt))
    tail = old.inputs[k0:]
    if len(tail) == 0:
        return None
    mc, sc = cfg.mppi, cfg.synthesis
    H, iters, k = len(tail), int(mc.iterations), int(sc.n_samples)
    gains = np.asarray(req.policy.gains, dtype=float)
    hold = int(gains.shape[0])
    key = (hold, H, int(req.t_proj), int(mc.batch), iters, k, float(mc.input_stdev), float(mc.temperature),
           float(sc.input_stdev), float(sc.r_running), float(dt), float(lim))
    cache = plan.__dict__.setdefault("_replan_graphs", {})
    parts = [np.clip(np.asarray(tail, dtype=float), -lim, lim), np.asarray(req.x, dtype=float), gains,
             np.asarray(old.states, dtype=float), np.asarray(old.inputs, dtype=float),
             np.asarray(mc.q_terminal, dtype=float), np.asarray(mc.x_perch, dtype=float),
             np.asarray(sc.state_stdev, dtype=float), np.asarray(sc.q_running, dtype=float),
             np.asarray(sc.q_final, dtype=float), np.array([old.t_start, float(req.t)])]
    plan.stage_fluid(req.fluid)
    if key not in cache:
        cache[key] = _ReplanGraph(torch, plan, dev, cfg, engine, hold, H, int(req.t_proj))
    g = cache[key]
    ints, traj, u, gain = g.run(parts, rng.seed, rng.iteration)
    rng.iteration += iters + 2
    st = ints[1 + max(iters, 1):1 + max(iters, 1) + k + 1]
    if ints[0] != 0 or (H and iters and mc.batch and np.any(ints[1:1 + iters] != 0)) or st[0] != 0:
        return None
    if int((st[1:] == 0).sum()) < 6 or ints[-1] != 0:
        return None
    nominal = NominalTrajectory(states=traj, inputs=u, dt=dt, t_start=t_new)
    return Policy(gains=gain, nominal=nominal, q_final=np.asarray(sc.q_final, dtype=float))


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
