"""TEST INFRASTRUCTURE ONLY: the unmodified reference package for the drop-in test.

``oracle/build_ref.sh`` stages ``/root/reference/pkg/src/perchsim`` (pure Python +
numpy) into the git-ignored ``oracle/_ref/pkg/`` so it travels to the GPU box.
:func:`load` imports it and :func:`install_backend` plugs a stepping module in
exactly where the reference's own compiled core goes
(``perchsim/_accel/__init__.py:14-18, 47-48``: ``backend_module()`` returns
``_core`` when the compiled backend is active) -- the swap
``tools/ref_trials.py`` makes with ``oracle/_ref``'s compiled core.
"""
from __future__ import annotations

import importlib
import os
import sys

_HERE = os.path.dirname(os.path.abspath(__file__))
PKG_DIR = os.path.join(_HERE, "_ref", "pkg")


def available() -> bool:
    return os.path.isfile(os.path.join(PKG_DIR, "perchsim", "_accel", "__init__.py"))


def load():
    """Import the staged reference ``perchsim`` (raises if it was never staged)."""
    if not available():
        raise ImportError(f"{PKG_DIR}/perchsim not staged: run oracle/build_ref.sh")
    if PKG_DIR not in sys.path:
        sys.path.insert(0, PKG_DIR)
    pkg = importlib.import_module("perchsim")
    assert os.path.dirname(pkg.__file__).startswith(PKG_DIR), pkg.__file__
    return pkg


def install_backend(module) -> None:
    """Make ``module`` the reference's compiled stepping core."""
    acc = importlib.import_module("perchsim._accel")
    acc._core, acc.HAVE_COMPILED, acc._active = module, True, "compiled"
