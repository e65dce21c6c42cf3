"""CPU tests: host-side API mirror, parameter ABI, boundary-system inverses, and
that the C-ABI library loads and exports every symbol include/vpm_b200.h declares."""
import ctypes
import math
import os
import re

import numpy as np
import pytest

from conftest import ROOT, golden


def test_pack_params_matches_reference_abi():
    from paper_2509_16079_b200 import config
    g = golden("c1_steps.npz")
    cfg = config.ExperimentConfig()
    cfg.vpm.particle_cap = 512
    ip, fp = config.pack_params(cfg.vpm, cfg.glider)
    np.testing.assert_array_equal(ip, g["iparams"])
    np.testing.assert_array_equal(fp, g["fparams"])


def test_config_validation_and_unknown_keys():
    from paper_2509_16079_b200 import config
    with pytest.raises(config.ConfigError, match="config.vpm.bogus"):
        config.config_from_dict({"vpm": {"bogus": 1}})
    with pytest.raises(config.ConfigError):
        config.config_from_dict({"vpm": {"particle_cap": 2}})
    cfg = config.config_from_dict({"mppi": {"batch": 4096, "horizon": 50}})
    assert cfg.mppi.batch == 4096 and len(cfg.config_hash()) == 16


def test_ring_injection_matches_reference_fixture():
    from paper_2509_16079_b200 import config, vpm
    sc = golden("scenario_C4.npz")
    cfg = config.VpmConfig(particle_cap=512)
    g = vpm.ring_circulation_for_speed(7.5, 0.28, 0.02)
    assert abs(g - 13.1949) < 1e-4  # SPEC.md:148-151 / SURVEY 8d
    fl = vpm.FluidState.empty(cfg)
    n = int(sc["n_wake"]) - 2
    for i in range(n):
        fl.append_particle(sc["wake_pos"][i], sc["wake_gamma"][i], int(sc["wake_age"][i]))
    fl = vpm.inject_ring(fl, vpm.RingDisturbance.from_speed([3.6, -0.1], 7.5, 0.28, 0.02, -1.0))
    assert (fl.ring_a, fl.ring_b) == (int(sc["ring_a"]), int(sc["ring_b"]))
    np.testing.assert_array_equal(fl.wake_pos[: fl.n_wake], sc["wake_pos"][: fl.n_wake])
    np.testing.assert_array_equal(fl.wake_gamma[: fl.n_wake], sc["wake_gamma"][: fl.n_wake])
    with pytest.raises(ValueError):
        vpm.inject_ring(fl, vpm.RingDisturbance.from_speed([0, 0], 7.5, 0.28, 0.02))
    c = fl.copy()
    assert c.equals(fl) and c is not fl
    c.wake_pos[0, 0] += 1.0
    assert not c.equals(fl)


def test_library_exports_every_declared_symbol():
    from paper_2509_16079_b200 import _lib
    hdr = open(os.path.join(ROOT, "include", "vpm_b200.h")).read()
    declared = set(re.findall(r"\b(vpm_[a-z0-9_]+)\s*\(", hdr))
    assert declared, "no declarations parsed"
    L = ctypes.CDLL(_lib.LIB_PATH)
    missing = [s for s in sorted(declared) if not hasattr(L, s)]
    assert not missing, missing
    assert set(_lib.EXPORTED) <= declared
    _lib.lib()  # full signature binding


def _reference_A(nb, l_chord, shed_off, lev_gain, theta, shed, rev, r=(0.3, -0.2)):
    """The boundary matrix as vpm.py:331-391 assembles it at an arbitrary pose."""
    f = np.array([math.cos(theta), math.sin(theta)])
    n = np.array([-math.sin(theta), math.cos(theta)])
    s = l_chord / nb
    col = np.array(r)[None, :] - np.outer(np.arange(nb + 1) * s, f)
    pan = col[:-1] - 0.5 * s * f
    lev, tev = col[0] + shed_off * f, col[-1] - shed_off * f
    cols = np.vstack([pan, lev, tev]) if shed else pan
    rows = (col[:nb] if rev else col[1:]) if shed else col[1:]
    ns = nb + 2 if shed else nb
    A = np.zeros((ns, ns))
    r0 = 1 if shed else 0
    for i, c in enumerate(rows):
        for j, p in enumerate(cols):
            d = c - p
            A[r0 + i, j] = (d[1] * n[0] - d[0] * n[1]) / (2 * math.pi * (d @ d))
    if shed:
        ec, ep = (nb + 1, nb - 1) if rev else (nb, 0)
        A[0, ec] = 1.0
        A[0, ep] = lev_gain
        A[nb + 1, :] = 1.0
    return A


@pytest.mark.parametrize("nb", [10, 4, 17])
def test_boundary_inverses_are_pose_invariant(nb):
    from paper_2509_16079_b200 import _lib, config
    v = config.VpmConfig(n_bound=nb)
    ip, fp = config.pack_params(v, config.GliderParams())
    S = nb + 2
    out = np.zeros(3 * S * S)
    assert _lib.lib().vpm_boundary_inverse(_lib.ptr(ip, _lib._I64), _lib.ptr(fp, _lib._D),
                                           _lib.ptr(out, _lib._D)) == 0
    rng = np.random.default_rng(nb)
    for var, (shed, rev) in enumerate([(False, False), (True, False), (True, True)]):
        ns = S if shed else nb
        Ainv = out[var * S * S: var * S * S + ns * ns].reshape(ns, ns)
        for theta in rng.uniform(-math.pi, math.pi, 5):
            A = _reference_A(nb, v.l_chord, v.shed_offset, v.lev_shed_gain, theta, shed, rev)
            np.testing.assert_allclose(A @ Ainv, np.eye(ns), atol=1e-9)


def test_backend_selection_has_no_cpu_path():
    from paper_2509_16079_b200 import _accel
    assert _accel.active_backend() == "cuda"
    _accel.set_backend("compiled")
    with pytest.raises(ValueError):
        _accel.set_backend("numpy")
    assert _accel.backend_module().__name__.endswith("_cuda")


def test_product_package_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2509_16079_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh")):
                src = open(os.path.join(dp, f)).read()
                assert "import oracle" not in src and "from oracle" not in src, f
                assert "liboracle" not in src and "_ref/" not in src, f


def test_symmetric_launch_shape_depends_on_the_cap_only():
    """The symmetric-pair sweep sums in an order fixed by its tile count, so every
    launch of a cap above 256 -- one step, a 513-row shard, a 4097-row iteration,
    C5's 16384 rows -- must get the same thread count (32 x ceil(cap / 128)) and at
    least four target slots per thread (vpm_capi.cu pick_shape).  Runs without a GPU
    (the SM count defaults to 148)."""
    import os
    from paper_2509_16079_b200.device import launch_shape
    for key in ("VPM_SHAPE", "VPM_SYM", "VPM_MAXREG"):
        assert key not in os.environ
    for cap in (257, 300, 512, 640, 1000, 1024, 2048):
        t_expect = 32 * ((cap + 127) // 128)
        shapes = {launch_shape(cap, 10, rows)[:2] for rows in (1, 65, 257, 513, 1025, 4097, 16384)}
        assert {t for t, _ in shapes} == {t_expect}, (cap, shapes)
        assert all(r >= 4 and t * r >= cap + 4 for t, r in shapes), (cap, shapes)
