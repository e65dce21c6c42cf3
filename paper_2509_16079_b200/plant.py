"""Device-resident fluids for the closed loop (nmpc.py:241-336 plant / observed wake).

The reference's control loop keeps two ``FluidState`` objects on the host and calls
``Engine.step`` (the plant, true flow) and ``Engine.fluid_step`` (the observed
wake around the measured state) every tick (nmpc.py:314-315); through the
stepping-module contract every call uploads the whole snapshot and downloads a fresh
one (rollout.py:81-98, _core.pyx:536-576).  :class:`DeviceWake` keeps one fluid in a
private ``vpm_plan`` whose snapshot the single-step kernel advances IN PLACE
(``vpm_plan_step``): the state and control go in by value as kernel arguments and
one 128-byte record (state, loads, wake size and ring indices, and optionally the
FP64 velocity at the pressure sensor) comes back per fluid, both fluids with one
stream synchronisation per tick.  The fluid is materialised on the host only when the loop needs it
(a replan request, a ring injection).

Results are bitwise those of the host-buffer path: the kernel forks the same FP64
snapshot values the host path would upload (the dump of the previous step).
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from ._lib import _D, addr, check, ptr
from .device import DevicePlan
from .vpm import FluidState

RECORD_BYTES = 128  # VPM_STEP_RECORD_BYTES: double x[7], fw[3], q[2]; int32 rc, n_wake, ring_a, ring_b, n_prev


class DeviceWake:
    """One fluid state resident on the device, stepped in place."""

    def __init__(self, engine, fluid: FluidState, stream=None):
        import torch
        self.cfg = engine.cfg
        self.plan = DevicePlan(engine.iparams, engine.fparams)
        self.plan.set_fluid(fluid)
        self.stream = stream if stream is not None else torch.cuda.Stream(torch.device("cuda", self.plan.device))
        self._rec = torch.zeros(RECORD_BYTES, dtype=torch.uint8, pin_memory=True)
        raw = self._rec.numpy()
        self._dbl = raw[:96].view(np.float64)   # x[7] fw[3] q[2]
        self._int = raw[96:116].view(np.int32)  # rc n_wake ring_a ring_b n_prev
        self._x = np.zeros(7)
        self._s2 = np.zeros(2)
        # fixed addresses, looked up once (the per-tick call passes plain integers)
        self._x_addr, self._s2_addr, self._rec_addr = addr(self._x), addr(self._s2), self._rec.data_ptr()
        self._stream_addr = self.stream.cuda_stream
        self.n_wake, self.ring_a, self.ring_b = fluid.n_wake, fluid.ring_a, fluid.ring_b
        self.rc = 0

    @property
    def disturbance(self):
        return None if self.ring_a < 0 else (self.ring_a, self.ring_b)

    def _s(self):
        return C.c_void_p(self._stream_addr)

    def step_async(self, x, u: float, integrate: bool, sensor=None, r_core: float = 0.0) -> None:
        """Queue one Engine.step (integrate) / fluid_step on the stream (state and
        control by value, one record copied back); with ``sensor`` the induced
        velocity there is evaluated on the stepped wake.  Read it with
        :meth:`record` after :meth:`sync`."""
        self._x[:] = x
        sp = None
        if sensor is not None:
            self._s2[:] = sensor
            sp = self._s2_addr
        check(_lib.lib().vpm_plan_step(self.plan.handle, self._x_addr, float(u), int(bool(integrate)), sp,
                                       float(r_core), self._rec_addr, self._stream_addr), "plan_step")

    def sync(self) -> None:
        check(_lib.lib().vpm_stream_sync(self._s()), "stream_sync")

    def record(self):
        """(rc, x (7,), fw (3,), q at the sensor (2,)) of the last queued step; also
        refreshes n_wake / ring indices."""
        d, i = self._dbl, self._int
        self.rc = int(i[0])
        self.n_wake, self.ring_a, self.ring_b = int(i[1]), int(i[2]), int(i[3])
        return self.rc, d[0:7].copy(), d[7:10].copy(), d[10:12].copy()

    def probe(self, target, r_core: float) -> np.ndarray:
        """Induced velocity (FP64) at one point from the current device wake (sync)."""
        self.sync()
        out = np.zeros(2)
        t = np.ascontiguousarray(target, dtype=float)
        check(_lib.lib().vpm_plan_probe(self.plan.handle, ptr(t, _D), float(r_core), ptr(out, _D)), "plan_probe")
        return out

    def download(self) -> FluidState:
        """The current device fluid as a host FluidState (reference layout)."""
        self.sync()
        flat = self.plan.download_fluid()
        f = FluidState.empty(self.cfg)
        (wp, wg, wa, n, ra, rb, pp, pg, m, pl, em) = flat
        f.wake_pos[:n], f.wake_gamma[:n], f.wake_age[:n] = wp[:n], wg[:n], wa[:n]
        f.n_wake, f.ring_a, f.ring_b = n, ra, rb
        f.prev_pos[:m], f.prev_gamma[:m], f.n_prev, f.prev_lev_gamma = pp[:m], pg[:m], m, pl
        f.unsteady_ema[:] = em
        return f

    def upload(self, fluid: FluidState) -> None:
        self.sync()
        self.plan.set_fluid(fluid)
        self.n_wake, self.ring_a, self.ring_b = fluid.n_wake, fluid.ring_a, fluid.ring_b
