"""Wake-index signature in Python (test infrastructure): the same function the
CUDA kernel (csrc/vpm_rollout.cuh ``wake_sig_*``) and the C oracle
(oracle/vpm_oracle.c ``sig_*``) evaluate, computed here from the reference's own
per-step outputs so the signature is pinned to the reference
(tests/golden/make_golden.py ``wake_sig``).

After every step's shed / merge / ring termination (_core.pyx:322-373) the chain
absorbs (wake size, ring-core indices, shed flag); the final wake contributes
sum_c mix(c, age_c).  Equal signatures mean identical shed steps, merges per step
and final index -> age order (remove_particle, _core.pyx:157-172)."""
from __future__ import annotations

M64 = (1 << 64) - 1


def mix(z: int) -> int:
    z = (z + 0x9E3779B97F4A7C15) & M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def step(h: int, n: int, ra: int, rb: int, shed: bool) -> int:
    key = (n & 0xFFFFFFFF) | (int(bool(shed)) << 31) | (((ra + 1) & 0xFFFF) << 32) | (((rb + 1) & 0xFFFF) << 48)
    return mix(h ^ key)


def signature(steps, ages) -> int:
    """steps: iterable of (n_wake, ring_a, ring_b, shed) after each step;
    ages: the final wake's ages in index order."""
    h = 0
    for n, ra, rb, shed in steps:
        h = step(h, int(n), int(ra), int(rb), bool(shed))
    s = 0
    for c, a in enumerate(ages):
        s = (s + mix(((c & 0xFFFFFFFF) << 32) | (int(a) & 0xFFFFFFFF))) & M64
    return mix(h ^ s)
