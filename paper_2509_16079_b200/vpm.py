"""Host-side fluid state containers and the gust-ring helpers.

Mirrors the data-structure half of ``perchsim/vpm.py`` (``FluidState``
vpm.py:144-234, ``VortexParticle``, ``RingDisturbance`` / ``inject_ring`` /
``ring_circulation_for_speed`` vpm.py:486-536): these are value-semantics host
snapshots that the planner forks onto the device.  All stepping physics of the
reference module (kernels, boundary solve, convection, shedding, merging, loads)
runs in the CUDA library, not here; ``induced_velocity`` / ``induced_velocity_at``
(vpm.py:93-128, the flow model of the NMPC pressure sensor) call the library's
FP64 device kernel.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .config import VpmConfig

TWO_PI = 2.0 * math.pi
KERNEL_REGULARIZED = "regularized"
KERNEL_SINGULAR = "singular"
_KERNEL_ID = {KERNEL_REGULARIZED: 0, KERNEL_SINGULAR: 1}


def induced_velocity_at(targets, positions, gammas, kernel: str = KERNEL_REGULARIZED,
                        r_core: float = 0.0) -> np.ndarray:
    """Velocity induced at each of the (m, 2) ``targets`` by point vortices at
    ``positions`` with circulations ``gammas`` (vpm.py:105-128), computed in FP64 on
    the device (``vpm_induced_velocity_host``).  Unknown kernels raise ValueError."""
    from . import _lib

    if kernel not in _KERNEL_ID:
        raise ValueError(f"unknown kernel {kernel!r}")
    tg = np.ascontiguousarray(np.atleast_2d(np.asarray(targets, dtype=np.float64)))
    out = np.zeros_like(tg)
    n = 0 if gammas is None else len(gammas)
    if n == 0 or len(tg) == 0:
        return out
    pos = np.ascontiguousarray(np.asarray(positions, dtype=np.float64).reshape(n, 2))
    gam = np.ascontiguousarray(np.asarray(gammas, dtype=np.float64))
    D = _lib._D
    _lib.check(_lib.lib().vpm_induced_velocity_host(_lib.ptr(pos, D), _lib.ptr(gam, D), n, _lib.ptr(tg, D),
                                                     len(tg), float(r_core), _KERNEL_ID[kernel],
                                                     _lib.ptr(out, D)), "induced_velocity")
    return out


def induced_velocity(positions, gammas, target, kernel: str = KERNEL_REGULARIZED,
                     r_core: float = 0.0) -> np.ndarray:
    """Summed velocity of many vortices at one target point (vpm.py:93-102)."""
    return induced_velocity_at(np.asarray(target, dtype=float).reshape(1, 2), positions, gammas,
                               kernel, r_core)[0]


@dataclass
class VortexParticle:
    position: np.ndarray
    circulation: float
    age: int = 0


class FluidState:
    """Wake particles (SoA, capacity cap+4) plus the previous bound row, its LEV
    strength and the unsteady-load filter state -- everything a step needs to be a
    pure function of (glider state, fluid state)."""

    __slots__ = ("wake_pos", "wake_gamma", "wake_age", "n_wake", "ring_a", "ring_b",
                 "prev_pos", "prev_gamma", "n_prev", "prev_lev_gamma", "unsteady_ema",
                 "particle_cap")

    def __init__(self, particle_cap: int, n_bound: int):
        slots = particle_cap + 4
        self.wake_pos = np.zeros((slots, 2))
        self.wake_gamma = np.zeros(slots)
        self.wake_age = np.zeros(slots, dtype=np.int64)
        self.n_wake = 0
        self.ring_a = -1
        self.ring_b = -1
        self.prev_pos = np.zeros((n_bound, 2))
        self.prev_gamma = np.zeros(n_bound)
        self.n_prev = 0
        self.prev_lev_gamma = 0.0
        self.unsteady_ema = np.zeros(n_bound)
        self.particle_cap = particle_cap

    @classmethod
    def empty(cls, cfg: VpmConfig) -> "FluidState":
        return cls(cfg.particle_cap, cfg.n_bound)

    def copy(self) -> "FluidState":
        out = FluidState.__new__(FluidState)
        for name in self.__slots__:
            v = getattr(self, name)
            setattr(out, name, v.copy() if isinstance(v, np.ndarray) else v)
        return out

    def equals(self, other: "FluidState") -> bool:
        n, m = self.n_wake, self.n_prev
        if (n, self.ring_a, self.ring_b, m, self.prev_lev_gamma) != (
                other.n_wake, other.ring_a, other.ring_b, other.n_prev, other.prev_lev_gamma):
            return False
        pairs = ((self.wake_pos[:n], other.wake_pos[:n]), (self.wake_gamma[:n], other.wake_gamma[:n]),
                 (self.wake_age[:n], other.wake_age[:n]), (self.prev_pos[:m], other.prev_pos[:m]),
                 (self.prev_gamma[:m], other.prev_gamma[:m]),
                 (self.unsteady_ema, other.unsteady_ema))
        return all(np.array_equal(a, b) for a, b in pairs)

    @property
    def disturbance(self):
        return None if self.ring_a < 0 else (self.ring_a, self.ring_b)

    def particles(self) -> list[VortexParticle]:
        return [VortexParticle(self.wake_pos[i].copy(), float(self.wake_gamma[i]),
                               int(self.wake_age[i])) for i in range(self.n_wake)]

    def append_particle(self, position, circulation: float, age: int = 0) -> int:
        i = self.n_wake
        if i >= self.wake_gamma.shape[0]:
            raise RuntimeError("wake buffer overflow")
        self.wake_pos[i] = position
        self.wake_gamma[i] = circulation
        self.wake_age[i] = age
        self.n_wake = i + 1
        return i

    def wake_circulation(self) -> float:
        return float(self.wake_gamma[: self.n_wake].sum())

    # flat 11-tuple of the stepping contract (rollout.py:59-62)
    def flat(self):
        return (self.wake_pos, self.wake_gamma, self.wake_age, self.n_wake, self.ring_a,
                self.ring_b, self.prev_pos, self.prev_gamma, self.n_prev, self.prev_lev_gamma,
                self.unsteady_ema)


def fluid_from_particles(particles, cfg: VpmConfig) -> FluidState:
    fluid = FluidState.empty(cfg)
    for p in particles:
        fluid.append_particle(np.asarray(p.position, dtype=float), p.circulation, p.age)
    return fluid


def ring_circulation_for_speed(speed: float, separation: float, r_core: float) -> float:
    """Pair strength that self-advects at ``speed`` under the smoothed kernel:
    v = G d / (2 pi sqrt(d^4 + rc^4))  (vpm.py:512-516)."""
    d = separation
    return speed * TWO_PI * math.sqrt(d ** 4 + r_core ** 4) / d


@dataclass
class RingDisturbance:
    """Planarised gust ring: a counter-rotating pair travelling along x."""

    center: np.ndarray
    speed: float
    separation: float
    r_core: float
    circulation: float
    direction: float = 1.0

    @classmethod
    def from_speed(cls, center, speed: float, separation: float, r_core: float,
                   direction: float = 1.0) -> "RingDisturbance":
        return cls(center=np.asarray(center, dtype=float), speed=speed, separation=separation,
                   r_core=r_core, circulation=ring_circulation_for_speed(speed, separation, r_core),
                   direction=direction)


def inject_ring(fluid: FluidState, ring: RingDisturbance) -> FluidState:
    """Append the ring pair (upper core first) and mark both as protected from
    merging (vpm.py:519-536).  For travel along +x the upper core is negative."""
    if fluid.disturbance is not None:
        raise ValueError("a ring disturbance is already active")
    out = fluid.copy()
    half = 0.5 * ring.separation
    sgn = 1.0 if ring.direction >= 0 else -1.0
    cx, cz = float(ring.center[0]), float(ring.center[1])
    out.ring_a = out.append_particle(np.array([cx, cz + half]), -sgn * ring.circulation, age=0)
    out.ring_b = out.append_particle(np.array([cx, cz - half]), sgn * ring.circulation, age=0)
    return out
