"""MPPI perching optimiser on the device (API of perchsim/mppi.py:19-84).

``optimize`` keeps the reference signature and random-number consumption: it
draws exactly what the reference draws from ``rng`` (one ``normal(0, 1, (K, H))``
block per iteration, each drawn while the device runs the previous iteration).
On the device each iteration is: one persistent rollout kernel over the K+1
candidates (row 0 = incumbent, rows 1..K = clip(u* + sigma * noise)) with the
terminal cost fused into its epilogue, one softmax-partial kernel and one combine
kernel (the same launches as the host-buffer C entry point
``vpm_mppi_optimize_host``, which takes all noise up front).

``terminal_cost``, ``terminal_cost_batch``, ``sample_controls`` and
``mppi_update`` are small host utilities on host arrays, kept for API parity;
``optimize`` does not use them.
"""

from __future__ import annotations

import numpy as np

from .config import MppiConfig
from .rollout import Engine
from .vpm import FluidState


def terminal_cost(x_final, cfg: MppiConfig) -> float:
    x = np.asarray(x_final, dtype=float)
    if not np.all(np.isfinite(x)):
        return float("inf")
    d = x - np.asarray(cfg.x_perch)
    return float(d @ (np.asarray(cfg.q_terminal) * d))


def terminal_cost_batch(finals, status, cfg: MppiConfig) -> np.ndarray:
    d = np.asarray(finals, dtype=float) - np.asarray(cfg.x_perch)[None, :]
    J = np.einsum("bi,i,bi->b", d, np.asarray(cfg.q_terminal, dtype=float), d)
    J[(np.asarray(status) != 0) | ~np.isfinite(J)] = np.inf
    return J


def sample_controls(mean, stdev: float, batch: int, rng: np.random.Generator,
                    u_limit: float) -> np.ndarray:
    mean = np.asarray(mean, dtype=float)
    return np.clip(mean[None, :] + rng.normal(0.0, 1.0, (batch, len(mean))) * stdev,
                   -u_limit, u_limit)


def mppi_update(controls, costs, temperature: float) -> np.ndarray:
    J = np.asarray(costs, dtype=float)
    ok = np.isfinite(J)
    if not ok.any():
        raise ValueError("all sampled rollouts failed (infinite cost)")
    w = np.where(ok, np.exp(-(J - J[ok].min()) / temperature), 0.0)
    return (w[:, None] * np.asarray(controls, dtype=float)).sum(axis=0) / w.sum()


def optimize(x0, fluid: FluidState, warm_start, cfg: MppiConfig, engine: Engine,
             rng: np.random.Generator, iterations: int | None = None) -> np.ndarray:
    """Iterated sample / rollout / reweight on the GPU; returns the final u*.

    Iteration i's noise is drawn on the host (exactly the reference's
    ``normal(0, 1, (K, H))`` call) while the device runs iteration i-1; the host
    synchronises once, at the end.  If an iteration finds every candidate failed,
    the reference raises after drawing that iteration's noise and no more: the
    generator is rewound and those draws replayed before ``ValueError`` is raised,
    so the caller's generator ends where the reference leaves it."""
    u_lim = engine.params.u_limit
    u = np.clip(np.asarray(warm_start, dtype=float).copy(), -u_lim, u_lim)
    iters = cfg.iterations if iterations is None else iterations
    H, K = len(u), int(cfg.batch)
    if H == 0 or iters == 0 or K == 0:
        return u
    import torch
    plan = engine_plan(engine)
    with plan.lock:
        return _optimize_locked(torch, plan, x0, fluid, u, cfg, rng, iters, H, K)


class DeviceNoise:
    """Performance mode for :func:`optimize` (and ``replan`` / ``build_policy``):
    pass ``DeviceNoise(seed)`` as ``rng`` and the control-perturbation noise is
    drawn on the device (counter-based Philox keyed by (seed, iteration, row),
    ``vpm_noise_philox``) instead of by numpy on the host -- no host RNG time and no
    host-to-device noise copy.  The numbers differ from numpy's, so reference parity
    uses a numpy Generator.  ``iteration`` advances by one per block drawn, across
    calls."""

    def __init__(self, seed: int, iteration: int = 0):
        self.seed = int(seed)
        self.iteration = int(iteration)


def _optimize_locked(torch, plan, x0, fluid, u, cfg, rng, iters, H, K):
    from .device import noise_philox
    devnoise = isinstance(rng, DeviceNoise)
    dev = torch.device("cuda", plan.device)
    plan.set_fluid(fluid)
    n_it = 0 if devnoise else K * H
    host = plan.staging(H + 21 + iters * n_it)
    hv = host.numpy()
    hv[:H] = u
    hv[H:H + 7] = np.asarray(x0, dtype=float)
    hv[H + 7:H + 14] = np.asarray(cfg.q_terminal, dtype=float)
    hv[H + 14:H + 21] = np.asarray(cfg.x_perch, dtype=float)
    head = host[:H + 21].to(dev, non_blocking=True)  # one pinned, non-blocking upload
    u_dev, x0d, q, xp = head[:H].clone(), head[H:H + 7], head[H + 7:H + 14], head[H + 14:H + 21]
    flags = torch.zeros(iters, dtype=torch.int32, device=dev)
    scratch = {"cost": torch.empty(K + 1, dtype=torch.float64, device=dev),
               "partial": torch.empty(H + 2, dtype=torch.float64, device=dev)}
    d_buf = torch.empty((K, H), dtype=torch.float64, device=dev) if devnoise else None
    saved = None if devnoise else rng.bit_generator.state
    for i in range(iters):
        if devnoise:
            d_noise = noise_philox(rng.seed, rng.iteration + i, d_buf)
        else:
            lo = H + 21 + i * n_it
            hv[lo:lo + n_it] = rng.normal(0.0, 1.0, (K, H)).ravel()
            d_noise = host[lo:lo + n_it].to(dev, non_blocking=True).view(K, H)
        scratch["flag"] = flags[i:i + 1]
        plan.mppi_iteration(x0d, u_dev, d_noise, cfg.input_stdev, K + 1, cfg.temperature, q, xp, scratch)
    if devnoise:
        rng.iteration += iters
    out = torch.cat([u_dev, flags.to(torch.float64)]).cpu().numpy()
    bad = np.nonzero(out[H:] != 0)[0]
    if bad.size:
        if not devnoise:  # leave the generator where the reference's raise leaves it
            rng.bit_generator.state = saved
            rng.normal(0.0, 1.0, (int(bad[0]) + 1, K, H))
        raise ValueError("all sampled rollouts failed (infinite cost)")
    return out[:H].copy()


def engine_plan(engine: Engine):
    """The device plan cached on an Engine (created on first use)."""
    from .device import DevicePlan
    plan = getattr(engine, "_device_plan", None)
    if plan is None:
        plan = DevicePlan(engine.iparams, engine.fparams)
        engine._device_plan = plan
    return plan
