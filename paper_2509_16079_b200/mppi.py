"""MPPI perching optimiser on the device (API of perchsim/mppi.py:19-84).

``optimize`` keeps the reference signature and random-number consumption: it
draws exactly what the reference draws from ``rng`` (one ``normal(0, 1, (K, H))``
block per iteration -- drawn here as one ``(iters, K, H)`` block, which numpy's
Generator fills identically) and hands everything to one C-ABI call,
``vpm_mppi_optimize_host``.  On the device each iteration is: one persistent
rollout kernel over the K+1 candidates (row 0 = incumbent, rows 1..K =
clip(u* + sigma * noise)) with the terminal cost fused into its epilogue, one
softmax-partial kernel and one combine kernel.

``terminal_cost``, ``terminal_cost_batch``, ``sample_controls`` and
``mppi_update`` are small host utilities on host arrays, kept for API parity;
``optimize`` does not use them.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from ._lib import _D, as_f64, check, ptr
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
    """Iterated sample / rollout / reweight on the GPU; returns the final u*."""
    u_lim = engine.params.u_limit
    u = np.clip(np.asarray(warm_start, dtype=float).copy(), -u_lim, u_lim)
    iters = cfg.iterations if iterations is None else iterations
    H, K = len(u), int(cfg.batch)
    if H == 0 or iters == 0 or K == 0:
        return u
    noise = as_f64(rng.normal(0.0, 1.0, (iters, K, H)))
    plan = engine_plan(engine)
    plan.set_fluid(fluid)
    q = as_f64(cfg.q_terminal)
    xp = as_f64(cfg.x_perch)
    x0a = as_f64(x0)
    check(_lib.lib().vpm_mppi_optimize_host(
        plan.handle, ptr(x0a, _D), ptr(u, _D), ptr(noise, _D), iters, K, H,
        float(cfg.input_stdev), float(cfg.temperature), ptr(q, _D), ptr(xp, _D)), "mppi.optimize")
    return u


def engine_plan(engine: Engine):
    """The device plan cached on an Engine (created on first use)."""
    from .device import DevicePlan
    plan = getattr(engine, "_device_plan", None)
    if plan is None:
        plan = DevicePlan(engine.iparams, engine.fparams)
        engine._device_plan = plan
    return plan
