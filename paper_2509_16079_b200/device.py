"""Device-resident planner plumbing: a ``vpm_plan`` handle plus torch-owned buffers.

PyTorch is used only for device memory, streams and ``torch.distributed``; all
compute is in ``libvpm_b200.so``.  :class:`DevicePlan` exposes the layer-2 C ABI
(``include/vpm_b200.h``) on CUDA tensors:

* :meth:`DevicePlan.batch` -- rollouts of an arbitrary row range of a candidate
  set, explicit controls or MPPI sampling, optional per-row start states,
  costs / diagnostics / trajectories (``vpm_plan_batch``);
* :meth:`DevicePlan.mppi_partial` / :func:`mppi_combine` -- the softmax update
  split into shard partials and a rank-ordered combine (``vpm_mppi_partial``,
  ``vpm_mppi_combine``), the pieces the multi-GPU driver puts an NCCL
  all-gather between (``sharding.py``);
* :meth:`DevicePlan.mppi_iteration` -- a whole single-device iteration.
"""

from __future__ import annotations

import ctypes as C
import threading

import numpy as np

from . import _lib
from ._lib import _D, _I32, _I64, VpmBatchOut, as_f64, as_i64, check, fluid_struct, ptr


def _torch():
    import torch
    return torch


def _p(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream(stream=None, device=None):
    """The launch stream: ``stream`` if given, else torch's current stream OF THE
    DEVICE the buffers live on (not of whatever device is current)."""
    torch = _torch()
    s = stream if stream is not None else torch.cuda.current_stream(device)
    return C.c_void_p(s.cuda_stream)


def _on(t):
    """Device guard for the plan-less entry points: kernels launch on the current
    device, so make it the device of ``t``."""
    return _torch().cuda.device(t.device)


def _need_f64(t, name, dim=None):
    torch = _torch()
    if not (t.is_cuda and t.dtype == torch.float64 and t.is_contiguous() and (dim is None or t.dim() == dim)):
        raise ValueError(f"{name} must be a contiguous CUDA float64 tensor"
                         + (f" of {dim} dimensions" if dim else ""))


class DevicePlan:
    """Owns one ``vpm_plan`` (inverse boundary matrices + fluid snapshot) on a device."""

    def __init__(self, iparams, fparams, device: int | None = None):
        self.iparams = as_i64(iparams)
        self.fparams = as_f64(fparams)
        if device is None:
            try:
                torch = _torch()
                device = torch.cuda.current_device() if torch.cuda.is_available() else 0
            except ImportError:
                device = 0
        self.device = int(device)
        L = _lib.lib()
        h = L.vpm_plan_create(ptr(self.iparams, _I64), ptr(self.fparams, _D), 0, 0, self.device)
        if not h:
            raise ValueError(f"vpm_plan_create: {_lib.last_error()}")
        self.handle = C.c_void_p(h)
        # the snapshot and the pinned staging buffer are per-plan state: host-side
        # sequences that set the snapshot and queue launches reading it (optimize,
        # replan, build_policy) hold this lock, so concurrent callers serialise
        self.lock = threading.RLock()
        self.nb = int(self.iparams[0])
        self.cap = int(self.iparams[1])

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and _lib._lib is not None:
            _lib._lib.vpm_plan_destroy(h)
            self.handle = None

    def staging(self, n: int):
        """Grow-only pinned host buffer of n float64 (async H2D of per-call draws).
        Callers synchronise before reusing it."""
        torch = _torch()
        buf = getattr(self, "_pinned", None)
        if buf is None or buf.numel() < n:
            buf = torch.empty(max(int(n), 1), dtype=torch.float64, pin_memory=True)
            self._pinned = buf
        return buf[:n]

    def set_fluid(self, fluid) -> None:
        flat = fluid.flat() if hasattr(fluid, "flat") else tuple(fluid)
        f, keep = fluid_struct(*flat)
        check(_lib.lib().vpm_plan_set_fluid(self.handle, C.byref(f)), "set_fluid")

    def stage_fluid(self, fluid) -> None:
        """Pack a snapshot into the pinned mirror without copying it up."""
        flat = fluid.flat() if hasattr(fluid, "flat") else tuple(fluid)
        f, keep = fluid_struct(*flat)
        check(_lib.lib().vpm_plan_stage_fluid(self.handle, C.byref(f)), "stage_fluid")

    def upload_fluid(self, stream=None) -> None:
        """Queue the pinned mirror's copy to the device snapshot (graph-capturable)."""
        check(_lib.lib().vpm_plan_upload_fluid(self.handle, _stream(stream, self.device)), "upload_fluid")

    # ---- rollouts -------------------------------------------------------------------
    def batch(self, x0, T: int, *, controls=None, ustar=None, noise=None, sigma: float = 0.0,
              row_begin: int = 0, rows: int | None = None, q=None, x_perch=None,
              record: bool = False, diagnostics: bool = False, stream=None, out=None):
        """Run rows [row_begin, row_begin + rows) on the device.  All tensor inputs
        are CUDA float64 tensors; returns a dict of CUDA tensors."""
        torch = _torch()
        dev = x0.device
        if rows is None:
            rows = controls.shape[0] if controls is not None else 1
        f64 = dict(dtype=torch.float64, device=dev)
        o = out if out is not None else {}
        if "status" not in o:
            o["status"] = torch.empty(rows, dtype=torch.int64, device=dev)
            o["finals"] = torch.empty(rows, 7, **f64)
            if q is not None:
                o["cost"] = torch.empty(rows, **f64)
            if record:
                o["trajs"] = torch.zeros(rows, T + 1, 7, **f64)
            if diagnostics:
                o["shed_mask"] = torch.zeros(rows, dtype=torch.int64, device=dev)
                o["n_final"] = torch.zeros(rows, dtype=torch.int32, device=dev)
                o["interactions"] = torch.zeros(rows, dtype=torch.int64, device=dev)
                o["shed_mask_hi"] = torch.zeros(rows, dtype=torch.int64, device=dev)
                o["wake_hash"] = torch.zeros(rows, dtype=torch.int64, device=dev)
        bo = VpmBatchOut(_p(o.get("status")), _p(o.get("finals")), _p(o.get("trajs")),
                         _p(o.get("cost")), _p(o.get("shed_mask")), _p(o.get("n_final")),
                         _p(o.get("interactions")), _p(o.get("shed_mask_hi")), _p(o.get("wake_hash")))
        stride = 7 if x0.dim() == 2 else 0
        check(_lib.lib().vpm_plan_batch(
            self.handle, _p(x0), stride, _p(controls), _p(ustar), _p(noise), float(sigma),
            int(row_begin), int(row_begin + rows), int(T), _p(q), _p(x_perch), int(bool(record)),
            C.byref(bo), _stream(stream, self.device)), "plan_batch")
        return o

    # ---- MPPI update ----------------------------------------------------------------
    def mppi_partial(self, cost, ustar, noise, sigma: float, temperature: float,
                     row_begin: int = 0, partial=None, stream=None):
        torch = _torch()
        T = int(ustar.shape[0])
        if partial is None:
            partial = torch.empty(T + 2, dtype=torch.float64, device=cost.device)
        check(_lib.lib().vpm_mppi_partial(
            self.handle, _p(cost), int(cost.shape[0]), int(row_begin), _p(ustar), _p(noise),
            float(sigma), T, float(temperature), _p(partial), _stream(stream, self.device)), "mppi_partial")
        return partial

    def mppi_iteration(self, x0, ustar, noise, sigma: float, B_total: int, temperature: float,
                       q, x_perch, scratch: dict, stream=None):
        """One single-device MPPI iteration, u* updated in place."""
        T = int(ustar.shape[0])
        check(_lib.lib().vpm_mppi_iteration(
            self.handle, _p(x0), _p(ustar), _p(noise), float(sigma), int(B_total), T,
            float(temperature), _p(q), _p(x_perch), _p(scratch["cost"]), _p(scratch["partial"]),
            _p(scratch["flag"]), 0, _stream(stream, self.device)), "mppi_iteration")

    # ---- replan pieces ------------------------------------------------------------------
    def project(self, x0, T: int, gains, states, inputs, t_start: float, t0: float,
                write_snapshot: bool = True, stream=None):
        """Closed-loop projection under a feedback policy (nmpc.py:88-103); returns
        (status (1,), final (1, 7)) device tensors."""
        torch = _torch()
        status = torch.zeros(1, dtype=torch.int64, device=x0.device)
        final = torch.empty(1, 7, dtype=torch.float64, device=x0.device)
        check(_lib.lib().vpm_plan_project(
            self.handle, _p(x0), int(T), _p(gains), _p(states), _p(inputs), int(gains.shape[0]),
            float(t_start), float(t0), _p(status), _p(final), int(bool(write_snapshot)),
            _stream(stream, self.device)), "plan_project")
        return status, final

    def project_dev(self, x0, T: int, gains, states, inputs, times, stream=None):
        """:meth:`project` with (t_start, t0) read from the device tensor ``times`` (2)
        when the kernel runs (CUDA-graph replay); writes the plan's snapshot."""
        torch = _torch()
        status = torch.zeros(1, dtype=torch.int64, device=x0.device)
        final = torch.empty(1, 7, dtype=torch.float64, device=x0.device)
        check(_lib.lib().vpm_plan_project_dev(
            self.handle, _p(x0), int(T), _p(gains), _p(states), _p(inputs), int(gains.shape[0]), _p(times),
            _p(status), _p(final), 1, _stream(stream, self.device)), "plan_project_dev")
        return status, final

    def cloud(self, x0, x0_noise, x0_scale, ustar, u_noise, sigma_u: float, stream=None):
        """Perturbed rollout cloud (policy.py:66-91): (status (K,), trajs (K, T+1, 7))."""
        torch = _torch()
        K, T = int(u_noise.shape[0]), int(ustar.shape[0])
        status = torch.empty(K, dtype=torch.int64, device=x0.device)
        trajs = torch.zeros(K, T + 1, 7, dtype=torch.float64, device=x0.device)
        check(_lib.lib().vpm_plan_cloud(
            self.handle, _p(x0), _p(x0_noise), _p(x0_scale), _p(ustar), _p(u_noise), float(sigma_u),
            K, T, _p(status), _p(trajs), _stream(stream, self.device)), "plan_cloud")
        return status, trajs

    def download_fluid(self):
        """The plan's current (device) snapshot as the reference's flat 11-tuple."""
        from ._lib import fluid_out, fluid_tuple
        fo, bufs = fluid_out(self.cap, self.nb)
        check(_lib.lib().vpm_plan_download_fluid(self.handle, C.byref(fo)), "download_fluid")
        return fluid_tuple(bufs)

    def timing(self, reset: int = 0):
        """(average rollout-kernel ms, launches) since the last reset; reset=1 starts
        recording CUDA events around every rollout launch, reset=-1 stops."""
        ms = np.zeros(1)
        n = np.zeros(1, dtype=np.int64)
        check(_lib.lib().vpm_plan_timing(self.handle, int(reset), ptr(ms, _D), ptr(n, _I64)),
              "plan_timing")
        return float(ms[0]), int(n[0])


def mppi_combine(partials, temperature: float, ustar, flag=None, stream=None):
    """Combine (W, T+2) gathered shard partials in rank order into ``ustar``."""
    W, ld = int(partials.shape[0]), int(partials.shape[1])
    _need_f64(partials, "partials", 2)
    _need_f64(ustar, "ustar", 1)
    with _on(ustar):
        check(_lib.lib().vpm_mppi_combine(_p(partials), W, ld - 2, float(temperature), _p(ustar),
                                          _p(flag), _stream(stream, ustar.device)), "mppi_combine")


def noise_philox(seed: int, iteration: int, out, row_begin: int = 0, stream=None):
    """Fill the CUDA float64 tensor ``out`` (rows, T) with rows [row_begin, row_begin
    + rows) of iteration ``iteration``'s device-drawn standard-normal noise
    (``vpm_noise_philox``: counter-based Philox keyed by (seed, iteration, row))."""
    _need_f64(out, "out", 2)  # the kernel writes rows x T doubles with row stride T
    rows, T = int(out.shape[0]), int(out.shape[1])
    with _on(out):
        check(_lib.lib().vpm_noise_philox(int(seed) & (2**64 - 1), int(iteration), int(row_begin), rows, T,
                                          _p(out), _stream(stream, out.device)), "noise_philox")
    return out


def noise_philox_dev(seed_iter, offset: int, out, row_begin: int = 0, stream=None):
    """:func:`noise_philox` with {seed, iteration} read from the device int64 tensor
    ``seed_iter`` (2) when the kernel runs (iteration + offset is drawn)."""
    _need_f64(out, "out", 2)
    rows, T = int(out.shape[0]), int(out.shape[1])
    with _on(out):
        check(_lib.lib().vpm_noise_philox_dev(_p(seed_iter), int(offset), int(row_begin), rows, T, _p(out),
                                              _stream(stream, out.device)), "noise_philox_dev")
    return out


def policy_fit(nom_x, nom_u, cloud_x, cloud_u, status, dt: float, q_running, r_running: float,
               q_final, stream=None):
    """Device regression + Riccati (policy.py:121-233) on device tensors; returns
    (a_cont, b_cont, a_disc, b_disc, gains, flag)."""
    torch = _torch()
    H, K = int(nom_u.shape[0]), int(cloud_u.shape[0])
    dev = nom_x.device
    # one uninitialised block, no fill kernels: the fit writes every entry of (ac, bc,
    # ad, bd) for every step, the Riccati every gain (on divergence it raises the flag
    # and the gains are not used); the flag itself must start at 0
    blk = torch.empty(H * (15 + 3 + 49 + 7 + 7), dtype=torch.float64, device=dev)
    ac, bc, ad, bd, g = (v.view(H, *sh) for v, sh in zip(
        torch.split(blk, [H * 15, H * 3, H * 49, H * 7, H * 7]), ((3, 5), (3,), (7, 7), (7,), (7,))))
    flag = torch.zeros(4, dtype=torch.int32, device=dev)
    with _on(nom_x):
        _policy_fit_call(nom_x, nom_u, cloud_x, cloud_u, status, K, H, dt, q_running, r_running, q_final,
                         ac, bc, ad, bd, g, flag, stream)
    return ac, bc, ad, bd, g, flag


def _policy_fit_call(nom_x, nom_u, cloud_x, cloud_u, status, K, H, dt, q_running, r_running, q_final,
                     ac, bc, ad, bd, g, flag, stream):
    check(_lib.lib().vpm_policy_fit(
        _p(nom_x), _p(nom_u), _p(cloud_x), _p(cloud_u), _p(status), K, H, float(dt), _p(q_running),
        float(r_running), _p(q_final), _p(ac), _p(bc), _p(ad), _p(bd), _p(g), _p(flag), 1, 1,
        _stream(stream, nom_x.device)), "policy_fit")


def launch_shape(cap: int, nb: int, rows: int):
    t, r, s = (np.zeros(1, np.int32) for _ in range(3))
    _lib.lib().vpm_launch_shape(int(cap), int(nb), int(rows), ptr(t, _I32), ptr(r, _I32), ptr(s, _I32))
    return int(t[0]), int(r[0]), int(s[0])


def fp32_peak_gflops(iters: int = 4096, mode: int = 0) -> float:
    """Measured pipe throughput: mode 0 FFMA GFLOP/s, 1 FFMA2 GFLOP/s, 2 MUFU.RSQ G ops/s."""
    return float(_lib.lib().vpm_fp32_peak_probe(int(iters), int(mode)))
