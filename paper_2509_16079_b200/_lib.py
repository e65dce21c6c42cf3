"""ctypes binding to ``lib/libvpm_b200.so`` (C ABI declared in ``include/vpm_b200.h``).

The library is built in-tree by :func:`build` (nvcc, ``-gencode
arch=compute_100a,code=sm_100a``) so the ``.so`` travels with the repository
snapshot to the GPU box.  There is no fallback: if the library cannot be loaded,
or no CUDA device is present, every entry point raises.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
LIB_PATH = os.environ.get("VPM_LIB") or os.path.join(PKG, "lib", "libvpm_b200.so")
SOURCES = [os.path.join(PKG, "csrc", "vpm_capi.cu"), os.path.join(PKG, "csrc", "vpm_rollout.cuh"),
           os.path.join(ROOT, "include", "vpm_b200.h")]
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-O3", "-std=c++17", "-fmad=false",
              "-shared", "-Xcompiler", "-fPIC"]

VPM_OK, VPM_ERR_CONFIG, VPM_ERR_CUDA, VPM_ERR_ALLFAIL, VPM_ERR_RANK, VPM_ERR_DIVERGED = (
    0, -1, -2, -3, -4, -5)


class CudaBackendError(RuntimeError):
    """The sm_100a library is missing, failed to load, or a CUDA call failed."""


def _stale() -> bool:
    if not os.path.exists(LIB_PATH):
        return True
    t = os.path.getmtime(LIB_PATH)
    return any(os.path.getmtime(s) > t for s in SOURCES if os.path.exists(s))


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile the CUDA library in place (cross-compiles without a GPU)."""
    if force or _stale():
        os.makedirs(os.path.dirname(LIB_PATH), exist_ok=True)
        nvcc = os.environ.get("NVCC", "nvcc")
        cmd = [nvcc, *NVCC_FLAGS, SOURCES[0], "-o", LIB_PATH + ".tmp"]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        subprocess.check_call(cmd)
        os.replace(LIB_PATH + ".tmp", LIB_PATH)
    return LIB_PATH


# ---- C structs (mirror include/vpm_b200.h) ----------------------------------------
_D = C.POINTER(C.c_double)
_I64 = C.POINTER(C.c_int64)
_I32 = C.POINTER(C.c_int32)
_U64 = C.POINTER(C.c_uint64)


# Pointer fields are declared c_void_p (the same ABI as the typed pointers of
# include/vpm_b200.h) so they take plain integer addresses: numpy's typed
# ``ctypes.data_as`` costs microseconds per pointer on the per-step host path.
class VpmFluid(C.Structure):
    _fields_ = [("wake_pos", C.c_void_p), ("wake_gamma", C.c_void_p), ("wake_age", C.c_void_p),
                ("n_wake", C.c_int32), ("ring_a", C.c_int32), ("ring_b", C.c_int32), ("prev_pos", C.c_void_p),
                ("prev_gamma", C.c_void_p), ("n_prev", C.c_int32), ("prev_lev", C.c_double), ("ema", C.c_void_p)]


class VpmFluidOut(C.Structure):
    _fields_ = [("wake_pos", C.c_void_p), ("wake_gamma", C.c_void_p), ("wake_age", C.c_void_p),
                ("scalars", C.c_void_p), ("prev_pos", C.c_void_p), ("prev_gamma", C.c_void_p),
                ("prev_lev", C.c_void_p), ("ema", C.c_void_p)]


class VpmBatchOut(C.Structure):
    _fields_ = [("status", C.c_void_p), ("finals", C.c_void_p), ("trajs", C.c_void_p),
                ("cost", C.c_void_p), ("shed_mask", C.c_void_p), ("n_final", C.c_void_p),
                ("interactions", C.c_void_p), ("shed_mask_hi", C.c_void_p), ("wake_hash", C.c_void_p)]


_lib = None
_lock = threading.Lock()


def lib():
    """Load (once) and return the library handle; raises CudaBackendError."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise CudaBackendError(
                f"{LIB_PATH} is not built; run __graft_entry__.build() (nvcc, sm_100a)")
        try:
            L = C.CDLL(LIB_PATH)
        except OSError as err:
            raise CudaBackendError(f"cannot load {LIB_PATH}: {err}") from err
        vp = C.c_void_p
        sig = {
            "vpm_step": (C.c_int, [vp, C.c_double, C.POINTER(VpmFluid), vp, vp, C.c_int, vp, vp,
                                   C.POINTER(VpmFluidOut)]),
            "vpm_rollout": (C.c_int64, [_D, _D, C.c_int, C.POINTER(VpmFluid), _I64, _D, _D,
                                        C.POINTER(VpmFluidOut)]),
            "vpm_batch_rollout": (C.c_int, [_D, _D, C.c_int, C.c_int, C.POINTER(VpmFluid), _I64, _D,
                                            C.c_int, C.c_int, _I64, _D, _D]),
            "vpm_batch_rollout_x0": (C.c_int, [_D, _D, C.c_int, C.c_int, C.POINTER(VpmFluid), _I64,
                                               _D, C.c_int, _I64, _D, _D]),
            "vpm_threads": (C.c_int, []),
            "vpm_last_error": (C.c_char_p, []),
            "vpm_plan_create": (vp, [_I64, _D, C.c_int, C.c_int, C.c_int]),
            "vpm_plan_destroy": (None, [vp]),
            "vpm_plan_set_fluid": (C.c_int, [vp, C.POINTER(VpmFluid)]),
            "vpm_plan_batch": (C.c_int, [vp, vp, C.c_int, vp, vp, vp, C.c_double, C.c_int, C.c_int,
                                         C.c_int, vp, vp, C.c_int, C.POINTER(VpmBatchOut), vp]),
            "vpm_mppi_partial": (C.c_int, [vp, vp, C.c_int, C.c_int, vp, vp, C.c_double, C.c_int,
                                           C.c_double, vp, vp]),
            "vpm_mppi_combine": (C.c_int, [vp, C.c_int, C.c_int, C.c_double, vp, vp, vp]),
            "vpm_noise_philox": (C.c_int, [C.c_uint64, C.c_uint64, C.c_int, C.c_int, C.c_int, vp, vp]),
            "vpm_mppi_iteration": (C.c_int, [vp, vp, vp, vp, C.c_double, C.c_int, C.c_int,
                                             C.c_double, vp, vp, vp, vp, vp, C.c_int, vp]),
            "vpm_mppi_optimize_host": (C.c_int, [vp, _D, _D, _D, C.c_int, C.c_int, C.c_int,
                                                 C.c_double, C.c_double, _D, _D]),
            "vpm_plan_timing": (C.c_int, [vp, C.c_int, _D, _I64]),
            "vpm_fp32_peak_probe": (C.c_double, [C.c_int, C.c_int]),
            "vpm_launch_shape": (C.c_int, [C.c_int, C.c_int, C.c_int, _I32, _I32, _I32]),
            "vpm_boundary_inverse": (C.c_int, [_I64, _D, _D]),
            "vpm_induced_velocity_host": (C.c_int, [_D, _D, C.c_int, _D, C.c_int, C.c_double, C.c_int, _D]),
            "vpm_policy_fit": (C.c_int, [vp, vp, vp, vp, vp, C.c_int, C.c_int, C.c_double, vp,
                                         C.c_double, vp, vp, vp, vp, vp, vp, vp, C.c_int, C.c_int,
                                         vp]),
            "vpm_build_policy_host": (C.c_int, [vp, _D, _D, C.c_int, _D, _D, C.c_int, C.c_double,
                                                _D, C.c_double, _D, _D, _D, _D, _D, _D, _I64, _D]),
            "vpm_policy_fit_host": (C.c_int, [_D, _D, C.c_int, _D, _D, _I64, C.c_int, C.c_double,
                                              _D, _D, _D, _D]),
            "vpm_tvlqr_host": (C.c_int, [_D, _D, C.c_int, _D, C.c_double, _D, _D]),
            "vpm_plan_project": (C.c_int, [vp, vp, C.c_int, vp, vp, vp, C.c_int, C.c_double,
                                           C.c_double, vp, vp, C.c_int, vp]),
            "vpm_plan_cloud": (C.c_int, [vp, vp, vp, vp, vp, vp, C.c_double, C.c_int, C.c_int, vp,
                                         vp, vp]),
            "vpm_plan_download_fluid": (C.c_int, [vp, C.POINTER(VpmFluidOut)]),
            "vpm_plan_step": (C.c_int, [vp, vp, C.c_double, C.c_int, vp, C.c_double, vp, vp]),
            "vpm_plan_probe": (C.c_int, [vp, _D, C.c_double, _D]),
            "vpm_stream_sync": (C.c_int, [vp]),
            "vpm_plan_stage_fluid": (C.c_int, [vp, C.POINTER(VpmFluid)]),
            "vpm_plan_upload_fluid": (C.c_int, [vp, vp]),
            "vpm_plan_project_dev": (C.c_int, [vp, vp, C.c_int, vp, vp, vp, C.c_int, vp, vp, vp, C.c_int, vp]),
            "vpm_noise_philox_dev": (C.c_int, [vp, C.c_uint64, C.c_int, C.c_int, C.c_int, vp, vp]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
        return _lib


EXPORTED = ("vpm_step", "vpm_rollout", "vpm_batch_rollout", "vpm_batch_rollout_x0", "vpm_threads",
            "vpm_last_error", "vpm_plan_create", "vpm_plan_destroy", "vpm_plan_set_fluid",
            "vpm_plan_batch", "vpm_mppi_partial", "vpm_mppi_combine", "vpm_noise_philox", "vpm_mppi_iteration",
            "vpm_mppi_optimize_host", "vpm_plan_timing", "vpm_fp32_peak_probe", "vpm_launch_shape",
            "vpm_boundary_inverse", "vpm_policy_fit", "vpm_build_policy_host",
            "vpm_policy_fit_host", "vpm_tvlqr_host", "vpm_plan_project", "vpm_plan_cloud",
            "vpm_plan_download_fluid", "vpm_induced_velocity_host", "vpm_plan_step", "vpm_plan_probe",
            "vpm_stream_sync", "vpm_plan_project_dev", "vpm_noise_philox_dev",
            "vpm_plan_stage_fluid", "vpm_plan_upload_fluid")


def last_error() -> str:
    return lib().vpm_last_error().decode(errors="replace")


def check(rc: int, what: str) -> int:
    """Map negative library returns to the reference's exception types."""
    if rc >= 0:
        return rc
    msg = f"{what}: {last_error()}"
    if rc == VPM_ERR_CONFIG:
        raise ValueError(msg)
    if rc == VPM_ERR_ALLFAIL:
        raise ValueError("all sampled rollouts failed (infinite cost)")
    if rc == VPM_ERR_RANK:
        from .policy import RankDeficientData
        raise RankDeficientData(last_error())
    if rc == VPM_ERR_DIVERGED:
        raise FloatingPointError(last_error())
    raise CudaBackendError(msg)


def ptr(a: np.ndarray, t):
    return a.ctypes.data_as(t)


def addr(a: np.ndarray) -> int:
    """Integer address of a contiguous array (for c_void_p arguments / fields)."""
    return a.ctypes.data


def as_f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def as_i64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int64)


def fluid_struct(wake_pos, wake_gamma, wake_age, n_wake, ring_a, ring_b, prev_pos, prev_gamma,
                 n_prev, prev_lev, ema):
    """Build a VpmFluid from the reference's flattened 11-tuple (rollout.py:59-62).
    Returns (struct, keepalive)."""
    keep = (as_f64(wake_pos), as_f64(wake_gamma), as_i64(wake_age), as_f64(prev_pos),
            as_f64(prev_gamma), as_f64(ema))
    f = VpmFluid(addr(keep[0]), addr(keep[1]), addr(keep[2]), int(n_wake), int(ring_a), int(ring_b),
                 addr(keep[3]), addr(keep[4]), int(n_prev), float(prev_lev), addr(keep[5]))
    return f, keep


def fluid_out(cap: int, nb: int, head: int = 0):
    """Output fluid buffers as views of ONE fresh float64 block (one address lookup):
    [head doubles | wake_pos 2(cap+4) | wake_gamma | wake_age (int64 view) | scalars
    (4 x int32 view) | prev_pos 2 nb | prev_gamma | prev_lev | ema]; ``bufs["head"]``
    is the caller's leading space, ``bufs["base"]`` the block's address."""
    c4 = cap + 4
    sizes = (head, 2 * c4, c4, c4, 2, 2 * nb, nb, 1, nb)
    offs = np.cumsum((0,) + sizes)
    block = np.zeros(int(offs[-1]))
    base = addr(block)
    o = [int(v) for v in offs]
    bufs = dict(head=block[o[0]:o[1]], wp=block[o[1]:o[2]].reshape(c4, 2), wg=block[o[2]:o[3]],
                wa=block[o[3]:o[4]].view(np.int64), sc=block[o[4]:o[5]].view(np.int32),
                pp=block[o[5]:o[6]].reshape(nb, 2), pg=block[o[6]:o[7]], pl=block[o[7]:o[8]],
                em=block[o[8]:o[9]], base=base)
    s = VpmFluidOut(*(base + 8 * o[i] for i in range(1, 9)))
    return s, bufs


def fluid_tuple(b):
    sc = b["sc"]
    return (b["wp"], b["wg"], b["wa"], int(sc[0]), int(sc[1]), int(sc[2]), b["pp"], b["pg"],
            int(sc[3]), float(b["pl"][0]), b["em"])
