"""TEST INFRASTRUCTURE ONLY: loader for the reference's own compiled stepping core.

``oracle/build_ref.sh`` compiles ``/root/reference/pkg/src/perchsim/_accel/_core.pyx``
(Cython + OpenMP, FP64) into ``oracle/_ref/_core*.so``.  That module has no
dependency on the rest of perchsim (numpy only), so it also loads on the GPU box,
where it is the ``--impl reference`` arm of bench.py and the ``"reference"``
kind of its ``cpu_baseline``.
"""

from __future__ import annotations

import glob
import importlib.util
import os

_HERE = os.path.dirname(os.path.abspath(__file__))


def path() -> str | None:
    hits = sorted(glob.glob(os.path.join(_HERE, "_ref", "_core*.so")))
    return hits[0] if hits else None


def load():
    """Return the reference ``_core`` module, or None when it was never built."""
    p = path()
    if p is None:
        return None
    spec = importlib.util.spec_from_file_location("_core", p)
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod
