"""TEST INFRASTRUCTURE ONLY: numpy restatement of the planner layer.

Restates, in FP64 numpy, the reference's MPPI optimiser
(``/root/reference/pkg/src/perchsim/mppi.py:19-84``) and sample-built TVLQR
controller (``policy.py:66-266``), driven by any object exposing the stepping
contract ``batch_rollout(...)`` (default: :mod:`oracle.core`).  Used by the
parity tests and by bench.py's CPU baseline; never by the product path.
"""

from __future__ import annotations

import numpy as np

from . import core as _core

DYN_ROWS = [4, 5, 6]          # policy.py:27
REG_COLS = [2, 3, 4, 5, 6]    # policy.py:28


def terminal_costs(finals, status, q, x_perch):
    """mppi.py:28-34: weighted squared distance to the perch; inf when failed."""
    d = np.asarray(finals, float) - np.asarray(x_perch, float)[None, :]
    J = (d * d) @ np.asarray(q, float)
    J = np.where((np.asarray(status) != 0) | ~np.isfinite(J), np.inf, J)
    return J


def candidates(u_star, noise, stdev, u_limit):
    """mppi.py:37-43 + :79: incumbent row 0, then clipped perturbed samples."""
    u_star = np.asarray(u_star, float)
    samp = np.clip(u_star[None, :] + np.asarray(noise, float) * stdev, -u_limit, u_limit)
    return np.concatenate([u_star[None, :], samp], axis=0)


def softmax_weights(J, temperature):
    """mppi.py:46-59 weights (unnormalised) with the J_min shift."""
    J = np.asarray(J, float)
    ok = np.isfinite(J)
    if not ok.any():
        raise ValueError("all sampled rollouts failed (infinite cost)")
    jmin = J[ok].min()
    return np.where(ok, np.exp(-(J - jmin) / temperature), 0.0)


def weighted_mean(controls, J, temperature):
    w = softmax_weights(J, temperature)
    return (w[:, None] * np.asarray(controls, float)).sum(axis=0) / w.sum()


def optimize(x0, flat_fluid, warm, noise_iters, iparams, fparams, *, stdev, temperature,
             q, x_perch, u_limit, stepper=_core, workers=0, trace=None):
    """mppi.py:62-84 with the per-iteration noise supplied explicitly
    (``noise_iters[i]`` is what ``rng.normal(0, 1, (K, H))`` returned)."""
    u = np.clip(np.asarray(warm, float).copy(), -u_limit, u_limit)
    for it in range(len(noise_iters)):
        cand = candidates(u, noise_iters[it], stdev, u_limit)
        status, finals, _ = stepper.batch_rollout(np.asarray(x0, float), cand, *flat_fluid,
                                                  iparams, fparams, False, workers)
        J = terminal_costs(finals, status, q, x_perch)
        if trace is not None:
            trace.append(dict(candidates=cand, status=status, finals=finals, costs=J,
                              weights=softmax_weights(J, temperature)))
        u = weighted_mean(cand, J, temperature)
    return u


def fit_sequence(nom_states, nom_inputs, states, inputs, ok, dt):
    """policy.py:121-171: per-step least squares of the acceleration rows on
    (theta, phi, v_x, v_z, omega, u) deviations with unexcited columns dropped;
    Euler discretisation with analytic kinematic rows."""
    nom_states = np.asarray(nom_states, float)
    nom_inputs = np.asarray(nom_inputs, float)
    S = np.asarray(states, float)[ok]
    U = np.asarray(inputs, float)[ok]
    H = len(nom_inputs)
    Ad = np.zeros((H, 7, 7))
    Bd = np.zeros((H, 7))
    dnom = (nom_states[1:] - nom_states[:-1]) / dt
    dsmp = (S[:, 1:] - S[:, :-1]) / dt
    for k in range(H):
        y = dsmp[:, k][:, DYN_ROWS] - dnom[k][DYN_ROWS]
        Z = np.concatenate([(S[:, k] - nom_states[k])[:, REG_COLS],
                            (U[:, k] - nom_inputs[k])[:, None]], axis=1)
        cn = np.linalg.norm(Z, axis=0)
        act = cn > 1e-10 * max(cn.max(), 1e-30)
        J = np.zeros((3, 6))
        if act.any():
            J[:, act] = np.linalg.lstsq(Z[:, act], y, rcond=None)[0].T
        Ac = np.zeros((7, 7))
        Bc = np.zeros(7)
        Ac[0, 4] = Ac[1, 5] = Ac[2, 6] = 1.0
        Bc[3] = 1.0
        Ac[np.ix_(DYN_ROWS, REG_COLS)] = J[:, :5]
        Bc[DYN_ROWS] = J[:, 5]
        Ad[k] = np.eye(7) + dt * Ac
        Bd[k] = dt * Bc
    return Ad, Bd


def riccati_gains(Ad, Bd, q_running, r_running, q_final):
    """policy.py:206-233: backward discrete Riccati recursion, (H, 7) gains."""
    Q = np.diag(np.asarray(q_running, float))
    S = np.diag(np.asarray(q_final, float))
    H = len(Ad)
    K = np.zeros((H, 7))
    for k in range(H - 1, -1, -1):
        A, b = Ad[k], Bd[k]
        Sb = S @ b
        h = (b @ S @ A) / float(r_running + b @ Sb)
        K[k] = h
        S = Q + A.T @ S @ A - np.outer(A.T @ Sb, h)
        S = 0.5 * (S + S.T)
        if not np.all(np.isfinite(S)):
            raise FloatingPointError(f"Riccati recursion diverged at step {k}")
    return K


def perturbed_cloud(nom_states, nom_inputs, flat_fluid, iparams, fparams, dx0_noise, du_noise,
                    state_stdev, input_stdev, u_limit, stepper=_core):
    """policy.py:66-91 with the two noise draws supplied explicitly."""
    x0s = np.asarray(nom_states, float)[0][None, :] + dx0_noise * np.asarray(state_stdev, float)
    U = np.clip(np.asarray(nom_inputs, float)[None, :] + du_noise * input_stdev, -u_limit, u_limit)
    d = stepper.batch_rollout_diag(x0s, U, *flat_fluid, iparams, fparams, record=True,
                                   per_rollout_x0=True)
    return d["trajs"], U, d["status"] == 0


def shard_partial(J, controls, temperature):
    """Per-shard softmax partial of the sharded update (paper_2509_16079_b200/sharding.py):
    (J_min_r, Z_r, S_r) over this shard's rows; J_min_r = inf when none is finite."""
    J = np.asarray(J, float)
    ok = np.isfinite(J)
    H = np.asarray(controls).shape[1]
    if not ok.any():
        return np.concatenate([[np.inf, 0.0], np.zeros(H)])
    jm = J[ok].min()
    w = np.where(ok, np.exp(-(J - jm) / temperature), 0.0)
    return np.concatenate([[jm, w.sum()], (w[:, None] * np.asarray(controls, float)).sum(axis=0)])


def combine_partials(parts, temperature):
    """Rank-ordered combine of gathered partials: rescale to the global J_min."""
    parts = np.asarray(parts, float)
    jm = parts[:, 0].min()
    if not np.isfinite(jm):
        raise ValueError("all sampled rollouts failed (infinite cost)")
    e = np.where(np.isfinite(parts[:, 0]), np.exp(-(parts[:, 0] - jm) / temperature), 0.0)
    return (e[:, None] * parts[:, 2:]).sum(axis=0) / (e * parts[:, 1]).sum()
