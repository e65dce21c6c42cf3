"""Stepping-backend plug point (mirrors perchsim/_accel/__init__.py:1-48).

The reference selects between its Cython/OpenMP core and a numpy backend.  This
package has exactly one backend -- the sm_100a CUDA library -- and no CPU
fallback: ``backend_module()`` always returns :mod:`._cuda`, whose entry points
raise :class:`~paper_2509_16079_b200._lib.CudaBackendError` when the library or a
GPU is unavailable.  ``PERCHSIM_BACKEND`` values other than ``auto``/``cuda``
(and the reference's alias ``compiled``) are rejected.
"""

import os

from . import _cuda

BACKENDS = ("cuda",)
_ALIASES = {"auto": "cuda", "": "cuda", "cuda": "cuda", "compiled": "cuda"}

_env = os.environ.get("PERCHSIM_BACKEND", "auto").lower()
if _env not in _ALIASES:
    raise ValueError(f"PERCHSIM_BACKEND={_env!r}: this package only provides the 'cuda' backend")
_active = "cuda"


def active_backend() -> str:
    return _active


def set_backend(name: str) -> None:
    """Accepts 'cuda' (or the reference alias 'compiled'); there is no CPU backend."""
    if _ALIASES.get(name) != "cuda":
        raise ValueError(f"unknown backend {name!r}: only 'cuda' is provided (no CPU fallback)")


def backend_module():
    return _cuda
