"""Drop-in proof: the UNMODIFIED reference package runs on the CUDA stepping module.

``oracle/build_ref.sh`` stages /root/reference/pkg/src/perchsim (git-ignored,
travels to the GPU box).  Here it is imported as is and
``paper_2509_16079_b200._accel._cuda`` is installed where the reference's own
compiled core goes (``perchsim/_accel/__init__.py:14-18, 47-48``; reached from
``rollout.py:56-57``).  The reference's own ``Engine.step``, ``mppi.optimize``,
``policy.build_policy`` and ``nmpc.control_loop`` then run every rollout through
the C ABI (``vpm_step`` / ``vpm_rollout`` / ``vpm_batch_rollout``) and are
compared with
  * this repository's mirror API on the same inputs (the stepping results are the
    same library calls: bitwise; reductions the reference does in numpy and the
    mirror on the device agree to FP64 rounding), and
  * the reference's golden vectors (tests/golden/, made with its numpy backend)
    within the tolerances stated in tests/test_gpu_parity.py.
"""
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, golden
from test_gpu_parity import X0, assert_close, fluid_from

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ref():
    import torch
    assert torch.cuda.is_available()
    from oracle import refpkg
    pkg = refpkg.load()
    from paper_2509_16079_b200._accel import _cuda
    refpkg.install_backend(_cuda)
    import perchsim._accel as acc
    assert acc.active_backend() == "compiled" and acc.backend_module() is _cuda
    return pkg


def _ref_fluid(perchsim, sc, cap):
    """The reference FluidState of a scenario fixture."""
    from perchsim import config as rc, vpm as rv
    f = rv.FluidState.empty(rc.VpmConfig(particle_cap=cap))
    n, m = int(sc["n_wake"]), int(sc["n_prev"])
    f.wake_pos[:n], f.wake_gamma[:n], f.wake_age[:n] = sc["wake_pos"][:n], sc["wake_gamma"][:n], sc["wake_age"][:n]
    f.n_wake, f.ring_a, f.ring_b = n, int(sc["ring_a"]), int(sc["ring_b"])
    f.prev_pos[:m], f.prev_gamma[:m], f.n_prev, f.prev_lev_gamma = sc["prev_pos"][:m], sc["prev_gamma"][:m], m, float(sc["prev_lev"])
    f.unsteady_ema[:] = sc["ema"]
    return f


def test_reference_engine_step_on_cuda(ref):
    """C1: 50 reference Engine.step calls (rollout.py:81-86) on the CUDA module."""
    from perchsim import config as rc, rollout as rr, vpm as rv
    from paper_2509_16079_b200 import config, rollout, vpm
    g = golden("c1_steps.npz")
    eng_r = rr.Engine(rc.VpmConfig(particle_cap=512), rc.GliderParams())
    eng_m = rollout.Engine(config.VpmConfig(particle_cap=512), config.GliderParams())
    np.testing.assert_array_equal(eng_r.fparams, g["fparams"])
    fr, fm = rv.FluidState.empty(eng_r.cfg), vpm.FluidState.empty(eng_m.cfg)
    xr, xm = X0.copy(), X0.copy()
    for t in range(50):
        okr, xr, fr, fwr = eng_r.step(xr, -15.0, fr)
        okm, xm, fm, fwm = eng_m.step(xm, -15.0, fm)
        assert okr and okm and fr.n_wake == fm.n_wake == g["n_wake_steps"][t]
        np.testing.assert_array_equal(xr, xm)
        np.testing.assert_array_equal(fwr, fwm)
        assert_close(xr, g["states"][t + 1], what=f"reference Engine.step state {t}")
    n = fr.n_wake
    np.testing.assert_array_equal(fr.wake_pos, fm.wake_pos)
    np.testing.assert_array_equal(fr.wake_age[:n], g["wake_age"][:n])
    assert_close(fr.wake_pos[:n], g["wake_pos"][:n], "wake_pos", what="reference Engine.step wake")
    # fluid_step and a single rollout with the final fluid returned (rollout.py:88-106)
    fr2, fw2, mw2 = eng_r.fluid_step(xr, fr)
    fm2, fwm2, mwm2 = eng_m.fluid_step(xm, fm)
    np.testing.assert_array_equal(fr2.wake_pos, fm2.wake_pos)
    assert mw2 == mwm2
    rcr, trr, flr = eng_r.rollout(X0, np.full(50, -15.0), rv.FluidState.empty(eng_r.cfg), record=True)
    assert rcr == 0 and flr.n_wake == 96
    assert_close(trr, g["states"], what="reference Engine.rollout")


def test_reference_mppi_optimize_on_cuda(ref):
    """C2: the reference's own mppi.optimize (mppi.py:62-84; 3 iterations, K=256,
    numpy PCG64 noise, numpy softmax update) with every batch on the CUDA module."""
    from perchsim import config as rc, mppi as rm, rollout as rr
    from paper_2509_16079_b200 import config, mppi, rollout
    g = golden("mppi_C2.npz")
    sc = golden("scenario_C2.npz")
    eng_r = rr.Engine(rc.VpmConfig(particle_cap=60), rc.GliderParams())
    u_r = rm.optimize(sc["x0"], _ref_fluid(ref, sc, 60), sc["warm"], rc.MppiConfig(batch=256, iterations=3, horizon=50),
                      eng_r, np.random.default_rng(int(g["seed"])))
    eng_m = rollout.Engine(config.VpmConfig(particle_cap=60), config.GliderParams())
    u_m = mppi.optimize(sc["x0"], fluid_from(sc, 60), sc["warm"], config.MppiConfig(batch=256, iterations=3, horizon=50),
                        eng_m, np.random.default_rng(int(g["seed"])))
    # same candidates, same rollouts; softmax reduction in numpy vs on the device
    np.testing.assert_allclose(u_r, u_m, rtol=1e-12, atol=1e-12)
    assert_close(u_r, g["u_star"], "u", what="reference mppi.optimize on CUDA vs golden")
    # one batch bitwise: the reference's Engine.batch vs the mirror's
    ctrl = np.clip(sc["warm"][None, :] + 2.0 * np.random.default_rng(3).normal(0, 1, (64, 50)), -15, 15)
    res_r = eng_r.batch(rr.RolloutRequest(x0=sc["x0"], fluid=_ref_fluid(ref, sc, 60), controls=ctrl, record=True))
    res_m = eng_m.batch(rollout.RolloutRequest(x0=sc["x0"], fluid=fluid_from(sc, 60), controls=ctrl, record=True))
    np.testing.assert_array_equal(res_r.status, res_m.status)
    np.testing.assert_array_equal(res_r.trajectories, res_m.trajectories)


def test_reference_build_policy_on_cuda(ref):
    """The reference's own policy.build_policy (policy.py:247-266): 64 sequential
    Engine.rollout calls through vpm_rollout, numpy lstsq regression and Riccati;
    against the mirror (one cloud launch + device regression / Riccati) and golden."""
    from perchsim import config as rc, policy as rp, rollout as rr
    from paper_2509_16079_b200 import config, policy, rollout
    g = golden("policy_C2.npz")
    sc = golden("scenario_C2.npz")
    eng_r = rr.Engine(rc.VpmConfig(particle_cap=60), rc.GliderParams())
    nom_r = rp.NominalTrajectory(states=g["nominal_states"], inputs=g["nominal_inputs"], dt=0.01)
    st_r, in_r, ok_r = rp.perturbed_rollouts(nom_r, _ref_fluid(ref, sc, 60), rc.SynthesisConfig(), eng_r,
                                             np.random.default_rng(int(g["seed"])))
    pol_r = rp.build_policy(nom_r, _ref_fluid(ref, sc, 60), rc.SynthesisConfig(), eng_r,
                            np.random.default_rng(int(g["seed"])))
    eng_m = rollout.Engine(config.VpmConfig(particle_cap=60), config.GliderParams())
    nom_m = policy.NominalTrajectory(states=g["nominal_states"], inputs=g["nominal_inputs"], dt=0.01)
    st_m, in_m, ok_m = policy.perturbed_rollouts(nom_m, fluid_from(sc, 60), config.SynthesisConfig(), eng_m,
                                                 np.random.default_rng(int(g["seed"])))
    pol_m = policy.build_policy(nom_m, fluid_from(sc, 60), config.SynthesisConfig(), eng_m,
                                np.random.default_rng(int(g["seed"])))
    np.testing.assert_array_equal(ok_r, ok_m)
    np.testing.assert_array_equal(ok_r, g["cloud_ok"])
    np.testing.assert_array_equal(st_r[ok_r], st_m[ok_m])  # 64 single rollouts == one cloud launch
    np.testing.assert_array_equal(in_r, in_m)
    np.testing.assert_allclose(pol_r.gains, pol_m.gains, rtol=1e-6, atol=1e-9)  # lstsq vs normal equations
    assert_close(st_r[ok_r], g["cloud_states"][ok_r], what="reference cloud on CUDA vs golden")
    assert_close(pol_r.gains, g["gains"], "gain", what="reference build_policy on CUDA vs golden")


def test_reference_control_loop_on_cuda(ref):
    """The reference's own closed-loop executive (nmpc.control_loop, nmpc.py:241-336:
    plant Engine.step + observed-wake fluid_step every tick, replans with
    mppi.optimize + build_policy) on the CUDA module, one trial per mode, against
    the same trials run on the reference's compiled core (ref_trials.json)."""
    from perchsim import nmpc as rn
    from perchsim.config import ExperimentConfig as RefCfg
    with open(os.path.join(GOLDEN, "ref_trials.json")) as fh:
        trials = json.load(fh)["trials"]
    out = {}
    for mode in ("no_disturbance", "uncompensated", "compensated"):
        rec = rn.control_loop(RefCfg(), mode, 0)
        gt = trials[f"{mode}/0"]
        assert len(rec.times) == gt["steps"], mode
        assert sum(e.accepted for e in rec.replans) == gt["replans_accepted"], mode
        assert (rec.failure is None) == (gt["failure"] is None)
        out[mode] = abs(rec.final_error - gt["final_error"])
        # closed loop over ~90 ticks and 7 replans: stated tolerance 1e-3 absolute (SI)
        np.testing.assert_allclose(rec.states[-1], gt["final_state"], rtol=0, atol=1e-3)
    print(json.dumps({"final_error_diff_m": out}))
    assert max(out.values()) <= 1e-4
