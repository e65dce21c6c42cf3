"""TEST INFRASTRUCTURE ONLY: ctypes binding to the FP64 C oracle (vpm_oracle.c).

Exposes the reference stepping-module contract
(``/root/reference/pkg/src/perchsim/_accel/_core.pyx:536-745``):

* ``step(x, u, *fluid11, iparams, fparams, integrate) -> (rc, x_new, fw, mw, fluid11)``
* ``rollout(x0, controls, *fluid11, iparams, fparams, record, return_fluid)
  -> (rc, traj_or_final, fluid11_or_None)``
* ``batch_rollout(x0, controls, *fluid11, iparams, fparams, record, workers)
  -> (status, finals, trajs_or_None)``
* ``omp_threads()``

plus :func:`batch_rollout_diag`, which also returns the shed bitmask, final wake
size and gate / ring-termination margins per rollout.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

_D = C.POINTER(C.c_double)
_I64 = C.POINTER(C.c_int64)
_I32 = C.POINTER(C.c_int32)
_U64 = C.POINTER(C.c_uint64)
_INT = C.POINTER(C.c_int)


def build() -> str:
    """Compile liboracle.so in place (gcc + OpenMP)."""
    src = os.path.join(_HERE, "vpm_oracle.c")
    if (not os.path.exists(_LIB_PATH)
            or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src)):
        subprocess.check_call(["make", "-s", "-C", _HERE, "liboracle.so"])
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = C.CDLL(_LIB_PATH)
        L.oracle_step.restype = C.c_int
        L.oracle_step.argtypes = [
            _D, C.c_double, _D, _D, _I64, C.c_int, C.c_int, C.c_int, _D, _D, C.c_int,
            C.c_double, _D, _I64, _D, C.c_int, _D, _D, _D, _D, _I64, _INT, _D, _D, _D, _D]
        L.oracle_batch_rollout.restype = C.c_int
        L.oracle_batch_rollout.argtypes = [
            _D, C.c_int, _D, C.c_int, C.c_int, _D, _D, _I64, C.c_int, C.c_int, C.c_int,
            _D, _D, C.c_int, C.c_double, _D, _I64, _D, _I64, _D, _D, _U64, _I32, _D, _D,
            _I64, _U64, _U64, C.c_int]
        L.oracle_rollout.restype = C.c_int64
        L.oracle_rollout.argtypes = [
            _D, _D, C.c_int, _D, _D, _I64, C.c_int, C.c_int, C.c_int, _D, _D, C.c_int,
            C.c_double, _D, _I64, _D, _D, _D, _D, _I64, _INT, _D, _D, _D, _D]
        L.oracle_threads.restype = C.c_int
        _lib = L
    return _lib


def _p(a, t):
    return None if a is None else a.ctypes.data_as(t)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


def _fluid_args(wake_pos, wake_gamma, wake_age, n_wake, ring_a, ring_b, prev_pos,
                prev_gamma, n_prev, prev_lev, ema):
    keep = (_f64(wake_pos), _f64(wake_gamma), _i64(wake_age), _f64(prev_pos),
            _f64(prev_gamma), _f64(ema))
    args = (_p(keep[0], _D), _p(keep[1], _D), _p(keep[2], _I64), int(n_wake), int(ring_a),
            int(ring_b), _p(keep[3], _D), _p(keep[4], _D), int(n_prev), float(prev_lev),
            _p(keep[5], _D))
    return keep, args


def _out_fluid(cap, nb):
    return dict(wp=np.zeros((cap + 4, 2)), wg=np.zeros(cap + 4),
                wa=np.zeros(cap + 4, dtype=np.int64), sc=np.zeros(4, dtype=np.intc),
                pp=np.zeros((nb, 2)), pg=np.zeros(nb), pl=np.zeros(1), em=np.zeros(nb))


def _out_args(o):
    return (_p(o["wp"], _D), _p(o["wg"], _D), _p(o["wa"], _I64), _p(o["sc"], _INT),
            _p(o["pp"], _D), _p(o["pg"], _D), _p(o["pl"], _D), _p(o["em"], _D))


def _out_tuple(o):
    sc = o["sc"]
    return (o["wp"], o["wg"], o["wa"], int(sc[0]), int(sc[1]), int(sc[2]), o["pp"], o["pg"],
            int(sc[3]), float(o["pl"][0]), o["em"])


def step(x, u, wake_pos, wake_gamma, wake_age, n_wake, ring_a, ring_b, prev_pos, prev_gamma,
         n_prev, prev_lev, ema, iparams, fparams, integrate):
    ip, fp = _i64(iparams), _f64(fparams)
    keep, fa = _fluid_args(wake_pos, wake_gamma, wake_age, n_wake, ring_a, ring_b, prev_pos,
                           prev_gamma, n_prev, prev_lev, ema)
    xs = _f64(x).copy()
    fw = np.zeros(2)
    mw = np.zeros(1)
    o = _out_fluid(int(ip[1]), int(ip[0]))
    rc = lib().oracle_step(_p(xs, _D), float(u), *fa, _p(ip, _I64), _p(fp, _D), int(bool(integrate)),
                           _p(fw, _D), _p(mw, _D), *_out_args(o))
    return rc, xs, fw, float(mw[0]), _out_tuple(o)


def rollout(x0, controls, wake_pos, wake_gamma, wake_age, n_wake, ring_a, ring_b, prev_pos,
            prev_gamma, n_prev, prev_lev, ema, iparams, fparams, record, return_fluid):
    ip, fp = _i64(iparams), _f64(fparams)
    keep, fa = _fluid_args(wake_pos, wake_gamma, wake_age, n_wake, ring_a, ring_b, prev_pos,
                           prev_gamma, n_prev, prev_lev, ema)
    u = _f64(controls).reshape(-1)
    T = len(u)
    xs = _f64(x0).copy()
    traj = np.zeros((T + 1, 7)) if record else None
    o = _out_fluid(int(ip[1]), int(ip[0]))
    rc = lib().oracle_rollout(_p(xs, _D), _p(u, _D), T, *fa, _p(ip, _I64), _p(fp, _D),
                              _p(traj, _D), *_out_args(o))
    out = traj if record else xs
    return int(rc), out, (_out_tuple(o) if return_fluid else None)


def batch_rollout_diag(x0, controls, wake_pos, wake_gamma, wake_age, n_wake, ring_a, ring_b,
                       prev_pos, prev_gamma, n_prev, prev_lev, ema, iparams, fparams,
                       record=False, workers=0, per_rollout_x0=False, per_step_n=False):
    """Batched rollouts plus diagnostics.  ``x0`` is (7,) or (B, 7) when
    ``per_rollout_x0``.  Returns a dict."""
    ip, fp = _i64(iparams), _f64(fparams)
    keep, fa = _fluid_args(wake_pos, wake_gamma, wake_age, n_wake, ring_a, ring_b, prev_pos,
                           prev_gamma, n_prev, prev_lev, ema)
    ctrl = _f64(controls)
    B, T = ctrl.shape
    x0a = _f64(x0)
    stride = 7 if per_rollout_x0 else 0
    out = dict(status=np.zeros(B, dtype=np.int64), finals=np.zeros((B, 7)),
               trajs=np.zeros((B, T + 1, 7)) if record else None,
               shed_mask=np.zeros(B, dtype=np.uint64), n_final=np.zeros(B, dtype=np.int32),
               gate_margin=np.zeros(B), ring_margin=np.zeros(B),
               n_steps=np.zeros((B, T), dtype=np.int64) if per_step_n else None,
               shed_mask_hi=np.zeros(B, dtype=np.uint64), wake_hash=np.zeros(B, dtype=np.uint64))
    lib().oracle_batch_rollout(
        _p(x0a, _D), stride, _p(ctrl, _D), B, T, *fa, _p(ip, _I64), _p(fp, _D),
        _p(out["status"], _I64), _p(out["finals"], _D), _p(out["trajs"], _D),
        _p(out["shed_mask"], _U64), _p(out["n_final"], _I32), _p(out["gate_margin"], _D),
        _p(out["ring_margin"], _D), _p(out["n_steps"], _I64), _p(out["shed_mask_hi"], _U64),
        _p(out["wake_hash"], _U64), int(workers))
    return out


def batch_rollout(x0, controls, wake_pos, wake_gamma, wake_age, n_wake, ring_a, ring_b,
                  prev_pos, prev_gamma, n_prev, prev_lev, ema, iparams, fparams, record,
                  workers):
    d = batch_rollout_diag(x0, controls, wake_pos, wake_gamma, wake_age, n_wake, ring_a, ring_b,
                           prev_pos, prev_gamma, n_prev, prev_lev, ema, iparams, fparams,
                           record=record, workers=workers)
    return d["status"], d["finals"], d["trajs"]


def omp_threads() -> int:
    return int(lib().oracle_threads())
