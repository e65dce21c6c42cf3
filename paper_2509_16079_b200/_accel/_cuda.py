"""The sm_100a stepping module: the reference's stepping contract on the GPU.

Same call signatures as the reference's compiled core
(``/root/reference/pkg/src/perchsim/_accel/_core.pyx:536-745``) -- flat FP64
arrays in, freshly allocated numpy arrays out -- implemented by the C ABI of
``libvpm_b200.so`` (``include/vpm_b200.h``: ``vpm_step``, ``vpm_rollout``,
``vpm_batch_rollout``, ``vpm_threads``).  Host<->device copies happen inside the
library; every rollout runs as one persistent CTA on the device.
"""

from __future__ import annotations

import numpy as np

from .. import _lib
from .._lib import _D, _I64, addr, as_f64, as_i64, check, fluid_out, fluid_struct, fluid_tuple, ptr


def step(x, u, wake_pos, wake_gamma, wake_age, n_wake, ring_a, ring_b, prev_pos, prev_gamma,
         n_prev, prev_lev, ema, iparams, fparams, integrate):
    """One coupled step.  Returns (status, x_new, fw, mw, fluid 11-tuple); _core.pyx:536-576."""
    ip, fp = as_i64(iparams), as_f64(fparams)
    f, keep = fluid_struct(wake_pos, wake_gamma, wake_age, n_wake, ring_a, ring_b, prev_pos,
                           prev_gamma, n_prev, prev_lev, ema)
    # x (7) | fw (2) | mw (1) lead the output fluid's block: one fresh allocation
    fo, bufs = fluid_out(int(ip[1]), int(ip[0]), head=10)
    h, base = bufs["head"], bufs["base"]
    h[:7] = as_f64(x).reshape(7)
    rc = check(_lib.lib().vpm_step(base, float(u), f, addr(ip), addr(fp), int(bool(integrate)), base + 56,
                                   base + 72, fo), "step")
    return rc, h[0:7], h[7:9], float(h[9]), fluid_tuple(bufs)


def rollout(x0, controls, wake_pos, wake_gamma, wake_age, n_wake, ring_a, ring_b, prev_pos,
            prev_gamma, n_prev, prev_lev, ema, iparams, fparams, record, return_fluid):
    """Open-loop rollout.  Returns (status, traj (T+1,7) or final (7,), fluid or None);
    _core.pyx:609-661."""
    ip, fp = as_i64(iparams), as_f64(fparams)
    f, keep = fluid_struct(wake_pos, wake_gamma, wake_age, n_wake, ring_a, ring_b, prev_pos,
                           prev_gamma, n_prev, prev_lev, ema)
    u = as_f64(controls).reshape(-1)
    T = int(u.shape[0])
    xs = as_f64(x0).copy()
    traj = np.zeros((T + 1, 7)) if record else None
    fo, bufs = fluid_out(int(ip[1]), int(ip[0])) if return_fluid else (None, None)
    st = _lib.lib().vpm_rollout(ptr(xs, _D), ptr(u, _D), T, f, ptr(ip, _I64), ptr(fp, _D),
                                ptr(traj, _D) if record else None, fo)
    check(int(st), "rollout")
    return int(st), (traj if record else xs), (fluid_tuple(bufs) if return_fluid else None)


def batch_rollout(x0, controls, wake_pos, wake_gamma, wake_age, n_wake, ring_a, ring_b,
                  prev_pos, prev_gamma, n_prev, prev_lev, ema, iparams, fparams, record, workers):
    """Batched rollouts.  Returns (status (B,), finals (B,7), trajs (B,T+1,7) or None);
    _core.pyx:664-714.  ``x0`` may be (7,) or, as an extension, (B, 7)."""
    ip, fp = as_i64(iparams), as_f64(fparams)
    f, keep = fluid_struct(wake_pos, wake_gamma, wake_age, n_wake, ring_a, ring_b, prev_pos,
                           prev_gamma, n_prev, prev_lev, ema)
    ctrl = as_f64(controls)
    if ctrl.ndim != 2:
        raise ValueError("controls must be (B, T)")
    B, T = ctrl.shape
    x0a = as_f64(x0)
    status = np.zeros(B, dtype=np.int64)
    finals = np.zeros((B, 7))
    trajs = np.zeros((B, T + 1, 7)) if record else None
    L = _lib.lib()
    tp = ptr(trajs, _D) if record else None
    if x0a.ndim == 2:
        rc = L.vpm_batch_rollout_x0(ptr(x0a, _D), ptr(ctrl, _D), B, T, f, ptr(ip, _I64), ptr(fp, _D),
                                    int(bool(record)), ptr(status, _I64), ptr(finals, _D), tp)
    else:
        rc = L.vpm_batch_rollout(ptr(x0a, _D), ptr(ctrl, _D), B, T, f, ptr(ip, _I64), ptr(fp, _D),
                                 int(bool(record)), int(workers), ptr(status, _I64),
                                 ptr(finals, _D), tp)
    check(rc, "batch_rollout")
    return status, finals, trajs


def omp_threads() -> int:
    """Concurrent rollouts resident on the device (the reference reports OpenMP threads)."""
    return int(_lib.lib().vpm_threads())
