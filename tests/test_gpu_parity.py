"""GPU parity: the sm_100a path (through the C ABI) against the reference's golden
vectors, the reference's own compiled core (oracle/_ref) and the FP64 CPU oracle on
identical inputs and identical noise.

Tolerances (stated; FP32 Biot-Savart sums and FP32 wake storage vs the
reference's float64).  Continuous quantities are checked as relative errors:

  * "elementwise":  |gpu - ref| <= rtol |ref| + atol
  * "normwise":     |gpu - ref| <= rtol max|ref| + atol, the max taken per physical
    component over the compared set (each state component over all rollouts /
    steps, u* over the horizon, each wake coordinate over the wake) -- a true
    relative error of the vector, defined where elementwise ratios are not
    (components cross zero: a final v_z of -0.045 m/s is reached along a
    trajectory where v_z spans +-3 m/s).

  quantity                              mode         rtol    atol
  glider states / finals / trajectories normwise     1e-4    1e-9
  wake positions / circulations         normwise     1e-4    1e-9
  wing force / moment                   normwise     1e-4    1e-9
  terminal costs                        elementwise  1e-4    0
  planned controls u*                   normwise     1e-4    0
  normalised MPPI weights               absolute     0       1e-4
  feedback gains (regression+Riccati)   normwise     1e-4    0

  Discrete decisions -- status, shed steps (128-bit mask), final wake size and the
  wake-index signature (per-step wake size / ring indices / shed flag + final
  index -> age order, tests/wake_sig.py) -- are exact, except on rollouts whose
  oracle-recorded gate or ring-termination margin is below GATE_DELTA /
  RING_DELTA (near-ties, counted and printed, never hidden).
"""
import numpy as np
import pytest

from conftest import flat_of, golden

pytestmark = pytest.mark.gpu

GATE_DELTA = 1e-5   # rad, | |aoa| - crit | and | |aoa| - pi/2 |
RING_DELTA = 1e-5   # intersection-parameter margin
X0 = np.array([0.0, 0.0, 0.3, 0.0, 7.0, 0.0, 0.0])
TOL = {  # kind: (mode, rtol, atol)
    "state": ("norm", 1e-4, 1e-9), "wake_pos": ("norm", 1e-4, 1e-9), "wake_gamma": ("norm", 1e-4, 1e-9),
    "fw": ("norm", 1e-4, 1e-9), "cost": ("elem", 1e-4, 0.0), "u": ("norm", 1e-4, 0.0),
    "weight": ("elem", 0.0, 1e-4), "gain": ("norm", 1e-4, 0.0)}


def assert_close(a, b, kind="state", what=""):
    """Relative-error check of TOL[kind]; normwise scales are taken per component
    (last axis) for arrays of 2+ dimensions, over the whole vector for 1-D ones."""
    mode, rtol, atol = TOL[kind]
    a, b = np.asarray(a, float), np.asarray(b, float)
    err = np.abs(a - b)
    if mode == "norm" and b.size:
        axes = tuple(range(b.ndim - 1)) if b.ndim >= 2 else None
        scale = np.max(np.abs(b), axis=axes, keepdims=b.ndim >= 2)
        bound = rtol * scale + atol + 0.0 * b
    else:
        bound = rtol * np.abs(b) + atol
    ok = err <= bound
    ratio = float(np.max(err / np.maximum(bound, 1e-300))) if err.size else 0.0
    rel = float(np.max(err / np.maximum(bound - atol, 1e-300) * rtol)) if (err.size and rtol > 0) else 0.0
    print(f"  {what or kind}: max |err| {err.max() if err.size else 0:.2e}, {mode}wise rel err "
          f"{rel:.2e}, max err/bound {ratio:.3f}")
    if not ok.all():
        i = np.unravel_index(np.argmax(err / np.maximum(bound, 1e-300)), np.shape(a))
        raise AssertionError(f"{what}: {int((~ok).sum())} entries off, worst at {i}: "
                             f"{a[i]} vs {b[i]} (bound {bound[i]:.3e}, {mode}wise rtol {rtol}, atol {atol})")


def mask128(lo, hi):
    return [int(np.uint64(l)) | (int(np.uint64(h)) << 64) for l, h in zip(lo, hi)]


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    assert torch.cuda.is_available()
    torch.cuda.set_device(0)
    return torch


def engine_for(iparams, fparams):
    from paper_2509_16079_b200 import config, rollout
    v = config.VpmConfig(particle_cap=int(iparams[1]))
    e = rollout.Engine(v, config.GliderParams())
    np.testing.assert_array_equal(e.fparams, fparams)
    return e


def fluid_from(g, cap):
    from paper_2509_16079_b200 import config, vpm
    f = vpm.FluidState.empty(config.VpmConfig(particle_cap=cap))
    (wp, wg, wa, n, ra, rb, pp, pg, m, pl, em) = flat_of(g)
    f.wake_pos[:n], f.wake_gamma[:n], f.wake_age[:n] = wp[:n], wg[:n], wa[:n]
    f.n_wake, f.ring_a, f.ring_b = n, ra, rb
    f.prev_pos[:m], f.prev_gamma[:m], f.n_prev, f.prev_lev_gamma = pp[:m], pg[:m], m, pl
    f.unsteady_ema[:] = em
    return f


# ------------------------------------------------------------------ golden vectors
def test_c1_step_sequence(torch_cuda):
    g = golden("c1_steps.npz")
    eng = engine_for(g["iparams"], g["fparams"])
    from paper_2509_16079_b200 import vpm
    fl = vpm.FluidState.empty(eng.cfg)
    x = X0.copy()
    for t in range(50):
        ok, x, fl, fw = eng.step(x, -15.0, fl)
        assert ok
        assert fl.n_wake == g["n_wake_steps"][t], t
        assert_close(x, g["states"][t + 1], what=f"state step {t}")
        assert_close(fw, g["fw"][t], "fw", what=f"fw step {t}")
    n = int(g["n_wake"])
    assert fl.n_wake == n == 96
    np.testing.assert_array_equal(fl.wake_age[:n], g["wake_age"][:n])
    assert_close(fl.wake_pos[:n], g["wake_pos"][:n], "wake_pos", what="wake_pos")
    assert_close(fl.wake_gamma[:n], g["wake_gamma"][:n], "wake_gamma", what="wake_gamma")


def test_c1_rollout_and_fluid(torch_cuda):
    g = golden("c1_steps.npz")
    eng = engine_for(g["iparams"], g["fparams"])
    from paper_2509_16079_b200 import vpm
    rc, traj, fl = eng.rollout(X0, np.full(50, -15.0), vpm.FluidState.empty(eng.cfg), record=True)
    assert rc == 0 and fl.n_wake == 96
    assert_close(traj, g["states"], what="traj")
    np.testing.assert_array_equal(fl.wake_age[:96], g["wake_age"][:96])


def test_batch_ring_golden(torch_cuda):
    g = golden("batch_ring.npz")
    eng = engine_for(g["iparams"], g["fparams"])
    from paper_2509_16079_b200 import rollout
    res = eng.batch(rollout.RolloutRequest(x0=X0, fluid=fluid_from(g, 128), controls=g["controls"],
                                           record=True))
    np.testing.assert_array_equal(res.status, g["status"])
    assert_close(res.trajectories, g["trajs"], what="trajs")


def test_fluid_step_matches_oracle(torch_cuda, oracle_core):
    sc = golden("scenario_C3.npz")
    eng = engine_for(sc["iparams"], sc["fparams"])
    fl = fluid_from(sc, 256)
    x = X0.copy()
    for k in range(3):
        fl_g, fw, mw = eng.fluid_step(x, fl)
        rc, _, fw_o, mw_o, flat_o = oracle_core.step(x, 0.0, *fl.flat(), eng.iparams, eng.fparams, False)
        assert rc == 0 and fl_g.n_wake == flat_o[3] and (fl_g.ring_a, fl_g.ring_b) == flat_o[4:6]
        n = fl_g.n_wake
        np.testing.assert_array_equal(fl_g.wake_age[:n], flat_o[2][:n])
        assert_close(fl_g.wake_pos[:n], flat_o[0][:n], "wake_pos", what="pos")
        assert_close(fl_g.wake_gamma[:n], flat_o[1][:n], "wake_gamma", what="gamma")
        assert_close(fw, fw_o, "fw", what="fw")
        fl = fl_g
        x[0] += 0.07


def test_mppi_C2_golden(torch_cuda):
    from paper_2509_16079_b200 import config, mppi
    g = golden("mppi_C2.npz")
    sc = golden("scenario_C2.npz")
    eng = engine_for(sc["iparams"], sc["fparams"])
    mcfg = config.MppiConfig(batch=256, iterations=3, horizon=50)
    u = mppi.optimize(sc["x0"], fluid_from(sc, 60), sc["warm"], mcfg, eng,
                      np.random.default_rng(int(g["seed"])))
    assert_close(u, g["u_star"], "u", what="u*")


def _device_iteration(torch, sc, K, seed, diagnostics=True):
    """One MPPI candidate batch through the device plan (C ABI layer 2)."""
    from paper_2509_16079_b200.device import DevicePlan
    plan = DevicePlan(sc["iparams"], sc["fparams"])
    plan.set_fluid(flat_of(sc))
    noise = np.random.default_rng(seed).normal(0.0, 1.0, (1, K, 50))
    dev = torch.device("cuda")
    f64 = lambda a: torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64), device=dev)
    q = f64([10, 10, 1, 0, 0.2, 0.2, 0.2])
    xp = f64([3.5, 0, np.pi / 4, 0, 0.5, -0.5, 0])
    out = plan.batch(f64(sc["x0"]), 50, ustar=f64(sc["warm"]), noise=f64(noise[0]), sigma=2.0,
                     rows=K + 1, q=q, x_perch=xp, diagnostics=diagnostics)
    torch.cuda.synchronize()
    return plan, noise, {k: v.cpu().numpy() for k, v in out.items()}


def _oracle_iteration(oracle_core, sc, noise):
    from oracle import planner
    cand = planner.candidates(sc["warm"], noise[0], 2.0, 15.0)
    d = oracle_core.batch_rollout_diag(sc["x0"], cand, *flat_of(sc), sc["iparams"], sc["fparams"])
    d["cost"] = planner.terminal_costs(d["finals"], d["status"], [10, 10, 1, 0, 0.2, 0.2, 0.2],
                                       [3.5, 0, np.pi / 4, 0, 0.5, -0.5, 0])
    d["cand"] = cand
    return d


def _check_decisions(gpu, ref, what):
    """Discrete decisions exact off near-ties: status, 128-bit shed mask, final wake
    size and the wake-index signature; returns the clean-and-successful row mask."""
    near = (ref["gate_margin"] < GATE_DELTA) | (ref["ring_margin"] < RING_DELTA)
    clean = ~near
    g_mask = np.array(mask128(gpu["shed_mask"], gpu["shed_mask_hi"]), dtype=object)
    r_mask = np.array(mask128(ref["shed_mask"], ref["shed_mask_hi"]), dtype=object)
    g_sig = gpu["wake_hash"].astype(np.uint64)
    differ = ((gpu["status"] != ref["status"]) | (g_mask != r_mask) | (gpu["n_final"] != ref["n_final"])
              | (g_sig != ref["wake_hash"]))
    B = len(ref["status"])
    print(f"{what}: {int(near.sum())} near-tie rollouts of {B} (margin < {GATE_DELTA:g}; "
          f"{int((differ & near).sum())} of them decided differently), "
          f"{int((ref['status'] != 0).sum())} failed, {int(clean.sum())} checked bit-exactly")
    np.testing.assert_array_equal(gpu["status"][clean], ref["status"][clean])
    assert (g_mask[clean] == r_mask[clean]).all(), "shed steps differ"
    np.testing.assert_array_equal(gpu["n_final"][clean], ref["n_final"][clean])
    np.testing.assert_array_equal(g_sig[clean], ref["wake_hash"][clean])
    assert not (differ & clean).any()
    return clean & (ref["status"] == 0)


@pytest.mark.parametrize("name,K,seed", [("scenario_C2.npz", 256, 11), ("scenario_C3.npz", 128, 12),
                                         ("scenario_C4.npz", 64, 13)])
def test_device_batch_vs_oracle_margin_aware(torch_cuda, oracle_core, name, K, seed):
    sc = golden(name)
    _, noise, gpu = _device_iteration(torch_cuda, sc, K, seed)
    ref = _oracle_iteration(oracle_core, sc, noise)
    ok = _check_decisions(gpu, ref, name)
    assert_close(gpu["finals"][ok], ref["finals"][ok], what="finals")
    assert_close(gpu["cost"][ok], ref["cost"][ok], "cost", what="cost")


@pytest.mark.parametrize("tag,name", [("c3", "scenario_C3.npz"), ("c4", "scenario_C4.npz"),
                                      ("c3long", "scenario_C3.npz")])
def test_wake_signature_vs_reference_golden(torch_cuda, tag, name):
    """The device kernel's wake-index signature against the one computed from the
    reference's own Engine.step sequence (tests/golden/wake_sig.npz): C3 / C4 MPPI
    candidates merging at the cap, and H = 100 rollouts (shed steps past 64)."""
    torch = torch_cuda
    from paper_2509_16079_b200.device import DevicePlan
    g = golden("wake_sig.npz")
    sc = golden(name)
    ctrl = g[tag + "_controls"]
    plan = DevicePlan(sc["iparams"], sc["fparams"])
    plan.set_fluid(flat_of(sc))
    dev = torch.device("cuda")
    out = plan.batch(torch.as_tensor(sc["x0"], device=dev), ctrl.shape[1],
                     controls=torch.as_tensor(ctrl, device=dev), rows=len(ctrl), diagnostics=True)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(out["status"].cpu().numpy(), g[tag + "_status"])
    np.testing.assert_array_equal(out["wake_hash"].cpu().numpy().astype(np.uint64), g[tag + "_sig"])
    assert_close(out["finals"].cpu().numpy(), g[tag + "_finals"], what=f"{tag} finals")


@pytest.mark.parametrize("name,K,seed", [("scenario_C3.npz", 1024, 31), ("scenario_C4.npz", 4096, 32)])
def test_full_iteration_vs_oracle(torch_cuda, oracle_core, name, K, seed):
    """Every candidate of a full C3 / C4 MPPI iteration (the headline batch, K+1
    rows, H=50, ring) on the same noise against
      * the reference's own compiled core (oracle/_ref, _core.pyx batch_rollout):
        status, finals, costs;
      * the FP64 C oracle (pinned to the reference, tests/test_oracle.py), which
        also records the per-rollout decision diagnostics: status, shed steps,
        final wake size and wake-index signature exact away from near-ties;
    and the MPPI update: normalised weights (mppi.py:46-59) within 1e-4 absolute,
    u* of the device update within 1e-4 relative of the oracle's."""
    import torch
    from oracle import planner, refcore
    from paper_2509_16079_b200.device import mppi_combine
    sc = golden(name)
    plan, noise, gpu = _device_iteration(torch, sc, K, seed)
    ref = _oracle_iteration(oracle_core, sc, noise)
    ok = _check_decisions(gpu, ref, f"{name} K={K}")
    assert_close(gpu["finals"][ok], ref["finals"][ok], what="finals vs oracle")
    assert_close(gpu["cost"][ok], ref["cost"][ok], "cost", what="cost vs oracle")
    # the reference's own compiled core on the same candidates
    rc = refcore.load()
    assert rc is not None, "oracle/_ref not built (oracle/build_ref.sh)"
    st_r, fin_r, _ = rc.batch_rollout(np.ascontiguousarray(sc["x0"]), np.ascontiguousarray(ref["cand"]),
                                      *flat_of(sc), sc["iparams"], sc["fparams"], False, 0)
    np.testing.assert_array_equal(st_r, ref["status"])  # FP64 vs FP64
    np.testing.assert_allclose(fin_r, ref["finals"], rtol=1e-9, atol=1e-11)
    J_r = planner.terminal_costs(fin_r, st_r, [10, 10, 1, 0, 0.2, 0.2, 0.2], [3.5, 0, np.pi / 4, 0, 0.5, -0.5, 0])
    clean = (ref["gate_margin"] >= GATE_DELTA) & (ref["ring_margin"] >= RING_DELTA)
    np.testing.assert_array_equal(gpu["status"][clean], st_r[clean])
    assert_close(gpu["finals"][ok], fin_r[ok], what="finals vs reference core")
    assert_close(gpu["cost"][ok], J_r[ok], "cost", what="cost vs reference core")
    # MPPI weights and u*
    fin = np.isfinite(J_r)
    def weights(J):
        w = np.where(np.isfinite(J), np.exp(-(J - J[np.isfinite(J)].min()) / 0.05), 0.0)
        return w / w.sum()
    w_g, w_r = weights(gpu["cost"]), weights(J_r)
    print(f"  weights: effective sample size {1.0 / np.sum(w_r ** 2):.1f}, max weight {w_r.max():.3f}")
    assert_close(w_g[fin], w_r[fin], "weight", what="normalised weights")
    dev = torch.device("cuda")
    us = torch.as_tensor(np.ascontiguousarray(sc["warm"]), device=dev)
    part = plan.mppi_partial(torch.as_tensor(gpu["cost"], device=dev), us,
                             torch.as_tensor(noise[0], device=dev), 2.0, 0.05)
    new = torch.empty_like(us)
    flag = torch.zeros(1, dtype=torch.int32, device=dev)
    mppi_combine(part.view(1, -1), 0.05, new, flag)
    torch.cuda.synchronize()
    assert flag.item() == 0
    u_gpu = new.cpu().numpy()
    np.testing.assert_allclose(u_gpu, planner.weighted_mean(ref["cand"], gpu["cost"], 0.05), rtol=1e-10,
                               atol=1e-12)
    assert_close(u_gpu, planner.weighted_mean(ref["cand"], J_r, 0.05), "u", what="u* vs reference core")


def test_mppi_update_vs_oracle(torch_cuda, oracle_core):
    """Softmax weights and u* from the device partial + combine kernels."""
    import torch
    from oracle import planner
    from paper_2509_16079_b200.device import mppi_combine
    sc = golden("scenario_C3.npz")
    K = 128
    plan, noise, gpu = _device_iteration(torch, sc, K, 21, diagnostics=False)
    ref = _oracle_iteration(oracle_core, sc, noise)
    dev = torch.device("cuda")
    cost = torch.as_tensor(gpu["cost"], device=dev)
    us = torch.as_tensor(np.ascontiguousarray(sc["warm"]), device=dev)
    nz = torch.as_tensor(noise[0], device=dev)
    part = plan.mppi_partial(cost, us, nz, 2.0, 0.05)
    new = torch.empty_like(us)
    flag = torch.zeros(1, dtype=torch.int32, device=dev)
    mppi_combine(part.view(1, -1), 0.05, new, flag)
    torch.cuda.synchronize()
    assert flag.item() == 0
    u_ref = planner.weighted_mean(ref["cand"], ref["cost"], 0.05)
    # same costs in -> FP64 update agrees to rounding
    u_same = planner.weighted_mean(ref["cand"], gpu["cost"], 0.05)
    np.testing.assert_allclose(new.cpu().numpy(), u_same, rtol=1e-10, atol=1e-12)
    assert_close(new.cpu().numpy(), u_ref, "u", what="u*")


@pytest.mark.parametrize("K,x0_mode", [(40, "scenario"), (128, "scenario"), (1024, "scenario"),
                                         (128, "blowup")])
def test_fused_iteration_equals_partial_plus_combine(torch_cuda, K, x0_mode):
    """vpm_mppi_iteration applies the W = 1 combine inside the softmax partial's
    finishing CTA: u*, the partial record and the sticky failure flag are bitwise what
    batch + vpm_mppi_partial + vpm_mppi_combine give -- for one chunk (K+1 <= 64),
    several chunks (last-CTA combine) and a batch whose every rollout fails (u* kept,
    flag raised)."""
    import torch
    from paper_2509_16079_b200.device import DevicePlan, mppi_combine
    sc = golden("scenario_C3.npz")
    plan = DevicePlan(sc["iparams"], sc["fparams"])
    plan.set_fluid(flat_of(sc))
    dev = torch.device("cuda")
    f64 = lambda a: torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64), device=dev)
    x0 = f64(sc["x0"] if x0_mode == "scenario" else [0.0, 0.0, 0.0, 0.0, 7.0, 0.0, 299.9])
    q, xp = f64([10, 10, 1, 0, 0.2, 0.2, 0.2]), f64([3.5, 0, np.pi / 4, 0, 0.5, -0.5, 0])
    noise = f64(np.random.default_rng(K).normal(0.0, 1.0, (K, 50)))
    us = f64(sc["warm"])
    scratch = {"cost": torch.empty(K + 1, dtype=torch.float64, device=dev),
               "partial": torch.empty(52, dtype=torch.float64, device=dev),
               "flag": torch.zeros(1, dtype=torch.int32, device=dev)}
    u_fused = us.clone()
    plan.mppi_iteration(x0, u_fused, noise, 2.0, K + 1, 0.05, q, xp, scratch)
    out = plan.batch(x0, 50, ustar=us, noise=noise, sigma=2.0, rows=K + 1, q=q, x_perch=xp)
    part = plan.mppi_partial(out["cost"], us, noise, 2.0, 0.05)
    u_sep, flag = us.clone(), torch.zeros(1, dtype=torch.int32, device=dev)
    mppi_combine(part.view(1, -1), 0.05, u_sep, flag)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(scratch["cost"].cpu().numpy(), out["cost"].cpu().numpy())
    np.testing.assert_array_equal(scratch["partial"].cpu().numpy(), part.cpu().numpy())
    np.testing.assert_array_equal(u_fused.cpu().numpy(), u_sep.cpu().numpy())
    assert int(scratch["flag"].item()) == int(flag.item()) == (1 if x0_mode == "blowup" else 0)
    if x0_mode == "blowup":
        assert not np.isfinite(out["cost"].cpu().numpy()).any()
        np.testing.assert_array_equal(u_fused.cpu().numpy(), sc["warm"])  # u* left unchanged
    else:
        assert not np.array_equal(u_fused.cpu().numpy(), sc["warm"])


def test_policy_C2_golden(torch_cuda):
    from paper_2509_16079_b200 import config, policy
    g = golden("policy_C2.npz")
    sc = golden("scenario_C2.npz")
    eng = engine_for(sc["iparams"], sc["fparams"])
    nom = policy.NominalTrajectory(states=g["nominal_states"], inputs=g["nominal_inputs"], dt=0.01)
    states, inputs, ok = policy.perturbed_rollouts(nom, fluid_from(sc, 60), config.SynthesisConfig(),
                                                   eng, np.random.default_rng(int(g["seed"])))
    np.testing.assert_array_equal(ok, g["cloud_ok"])
    assert_close(states[ok], g["cloud_states"][ok], what="cloud")
    pol = policy.build_policy(nom, fluid_from(sc, 60), config.SynthesisConfig(), eng,
                              np.random.default_rng(int(g["seed"])))
    assert_close(pol.gains, g["gains"], "gain", what="gains")


def test_policy_kernels_on_reference_cloud(torch_cuda):
    """The device regression + Riccati on the reference's own perturbed cloud
    (identical inputs): FP64 normal equations with column scaling vs LAPACK gelsd."""
    from paper_2509_16079_b200 import policy
    g = golden("policy_C2.npz")
    nom = policy.NominalTrajectory(states=g["nominal_states"], inputs=g["nominal_inputs"], dt=0.01)
    # the reference's inputs for the cloud: clip(nominal + du * 0.5)
    U = np.clip(g["nominal_inputs"][None, :] + g["du"] * 0.5, -15, 15)
    seq = policy.estimate_linear_sequence(nom, g["cloud_states"], U, g["cloud_ok"], 0.01)
    np.testing.assert_allclose(seq.a_discrete, g["a_discrete"], rtol=1e-7, atol=1e-9)
    np.testing.assert_allclose(seq.b_discrete, g["b_discrete"], rtol=1e-7, atol=1e-9)
    K = policy.tvlqr_backward(g["a_discrete"], g["b_discrete"], [0.1, 0.1, 5.0, 0.1, 0.1, 0.1, 5.0],
                              0.01, [400.0, 400.0, 10.0, 1.0, 1.0, 1.0, 1.0])
    np.testing.assert_allclose(K, g["gains"], rtol=1e-9, atol=1e-9)
    with pytest.raises(FloatingPointError):
        policy.tvlqr_backward(g["a_discrete"] * 1e200, g["b_discrete"], [1] * 7, 0.01, [1] * 7)


def test_replan_on_device_matches_reference(torch_cuda):
    """nmpc.replan (project 10 closed-loop steps, 3 MPPI iterations K=256 over the
    67-step tail, nominal rollout, policy) against the reference run with the same
    bootstrap policy and rng seed (tests/golden/make_golden.py replan)."""
    from paper_2509_16079_b200 import config, replan, rollout, vpm
    from paper_2509_16079_b200.policy import NominalTrajectory, Policy
    g = golden("nmpc_replan.npz")
    cfg = config.ExperimentConfig()
    eng = rollout.Engine.from_config(cfg)
    pol = Policy(gains=g["boot_gains"], nominal=NominalTrajectory(g["boot_states"], g["boot_inputs"], 0.01))
    x0 = np.asarray(cfg.scenario.x0, dtype=float)
    fl0 = vpm.FluidState.empty(cfg.vpm)
    xp, flp, tp = replan.project_forward(pol, x0, fl0, 0.0, 10, eng)
    assert tp == g["proj_t"] and flp.n_wake == int(g["proj_n_wake"])
    assert_close(xp, g["proj_x"], what="projected state")
    np.testing.assert_array_equal(flp.wake_age[: flp.n_wake], g["proj_wake_age"])
    assert_close(flp.wake_pos[: flp.n_wake], g["proj_wake_pos"], "wake_pos", what="projected wake")
    new = replan.replan(replan.ReplanRequest(x=x0, fluid=fl0, policy=pol, t=0.0, t_proj=10), cfg, eng,
                        np.random.default_rng(1))
    assert new is not None and new.t_start == g["new_t_start"]
    assert_close(new.nominal.inputs, g["new_inputs"], "u", what="replanned u*")
    assert_close(new.nominal.states, g["new_states"], "state", what="replanned nominal")
    assert_close(new.gains, g["new_gains"], "gain", what="replanned gains")


def test_replan_leaves_the_generator_where_the_reference_does(torch_cuda):
    """The replan draws every random number up front; the caller's generator must
    still end exactly where the reference's would (nmpc.py:118-134): after a
    success, iters x (K, H) MPPI noises then the cloud's (64, 7) and (64, H); after a
    failed projection, untouched."""
    from paper_2509_16079_b200 import config, replan, rollout, vpm
    from paper_2509_16079_b200.policy import NominalTrajectory, Policy
    g = golden("nmpc_replan.npz")
    cfg = config.ExperimentConfig()
    eng = rollout.Engine.from_config(cfg)
    pol = Policy(gains=g["boot_gains"], nominal=NominalTrajectory(g["boot_states"], g["boot_inputs"], 0.01))
    x0 = np.asarray(cfg.scenario.x0, dtype=float)
    fl0 = vpm.FluidState.empty(cfg.vpm)
    rng, twin = np.random.default_rng(11), np.random.default_rng(11)
    new = replan.replan(replan.ReplanRequest(x=x0, fluid=fl0, policy=pol, t=0.0, t_proj=10), cfg, eng, rng)
    assert new is not None
    H = new.nominal.horizon
    for _ in range(cfg.mppi.iterations):
        twin.normal(0.0, 1.0, (cfg.mppi.batch, H))
    twin.normal(0.0, 1.0, (cfg.synthesis.n_samples, 7))
    twin.normal(0.0, 1.0, (cfg.synthesis.n_samples, H))
    assert rng.bit_generator.state == twin.bit_generator.state
    # the nominal of the fused nominal+cloud launch is the plain rollout of u*
    rc, traj, _ = eng.rollout(new.nominal.states[0], new.nominal.inputs, replan.project_forward(
        pol, x0, fl0, 0.0, 10, eng)[1], record=True)
    assert rc == 0
    np.testing.assert_array_equal(traj, new.nominal.states)
    # a projection that leaves the envelope rejects the replan without drawing
    bad = x0.copy()
    bad[6] = 400.0
    before = rng.bit_generator.state
    assert replan.replan(replan.ReplanRequest(x=bad, fluid=fl0, policy=pol, t=0.0, t_proj=10), cfg, eng,
                         rng) is None
    assert rng.bit_generator.state == before


# ------------------------------------------------------------------ full-size properties
def test_c4_full_batch_properties(torch_cuda, oracle_core):
    """K=4096, H=50, N=512 + ring: deterministic, row-independent (batch ==
    sub-batch), finite, and a random subset matches the oracle."""
    torch = torch_cuda
    sc = golden("scenario_C4.npz")
    K = 4096
    plan, noise, a = _device_iteration(torch, sc, K, 5)
    _, _, b = _device_iteration(torch, sc, K, 5)
    for k in ("status", "finals", "cost", "shed_mask", "shed_mask_hi", "n_final", "wake_hash"):
        np.testing.assert_array_equal(a[k], b[k])
    assert np.all(a["n_final"] <= 512) and np.all(a["n_final"] >= 500)
    # a 33-row slice computed alone is bitwise identical to the same rows of the full batch
    from paper_2509_16079_b200.device import DevicePlan
    dev = torch.device("cuda")
    f64 = lambda v: torch.as_tensor(np.ascontiguousarray(v, dtype=np.float64), device=dev)
    q = f64([10, 10, 1, 0, 0.2, 0.2, 0.2])
    xp = f64([3.5, 0, np.pi / 4, 0, 0.5, -0.5, 0])
    sub = plan.batch(f64(sc["x0"]), 50, ustar=f64(sc["warm"]), noise=f64(noise[0]), sigma=2.0,
                     row_begin=2000, rows=33, q=q, x_perch=xp)
    np.testing.assert_array_equal(sub["finals"].cpu().numpy(), a["finals"][2000:2033])
    # oracle on 24 random rows
    rows = np.random.default_rng(0).choice(K + 1, 24, replace=False)
    from oracle import planner
    cand = planner.candidates(sc["warm"], noise[0], 2.0, 15.0)[rows]
    d = oracle_core.batch_rollout_diag(sc["x0"], cand, *flat_of(sc), sc["iparams"], sc["fparams"])
    sub_a = {k: v[rows] for k, v in a.items()}
    ok = _check_decisions(sub_a, d, "C4 random rows")
    assert_close(sub_a["finals"][ok], d["finals"][ok], what="finals")


# ------------------------------------------------------------------ edge cases
def test_zero_horizon_and_empty_batch(torch_cuda):
    from paper_2509_16079_b200 import config, rollout, vpm
    eng = rollout.Engine(config.VpmConfig(), config.GliderParams())
    fl = vpm.FluidState.empty(eng.cfg)
    rc, traj, fo = eng.rollout(X0, np.zeros(0), fl, record=True)
    assert rc == 0 and traj.shape == (1, 7) and np.array_equal(traj[0], X0) and fo.n_wake == 0
    res = eng.batch(rollout.RolloutRequest(x0=X0, fluid=fl, controls=np.zeros((0, 5))))
    assert res.status.shape == (0,)


@pytest.mark.parametrize("nb,cap", [(4, 4), (10, 8), (17, 40), (33, 100), (10, 300)])
def test_odd_configs_vs_oracle(torch_cuda, oracle_core, nb, cap):
    """Small caps (merging every step, ring protected), nb beyond a warp, tile overflow."""
    from paper_2509_16079_b200 import config, rollout, vpm
    v = config.VpmConfig(n_bound=nb, particle_cap=cap)
    eng = rollout.Engine(v, config.GliderParams())
    fl = vpm.FluidState.empty(v)
    fl = vpm.inject_ring(fl, vpm.RingDisturbance.from_speed([0.8, -0.05], 7.5, 0.28, 0.02, -1.0))
    rng = np.random.default_rng(nb * 1000 + cap)
    ctrl = np.clip(-8.0 + 4.0 * rng.normal(0, 1, (16, 40)), -15, 15)
    res = eng.batch(rollout.RolloutRequest(x0=X0, fluid=fl, controls=ctrl, record=True))
    d = oracle_core.batch_rollout_diag(X0, ctrl, *fl.flat(), eng.iparams, eng.fparams, record=True)
    clean = (d["gate_margin"] >= GATE_DELTA) & (d["ring_margin"] >= RING_DELTA)
    np.testing.assert_array_equal(res.status[clean], d["status"][clean])
    ok = clean & (d["status"] == 0)
    # Conditioning: the ring is injected 0.8 m ahead, its cores (r_c = 0.02) sweep
    # past the plate and small caps merge every step, so the FP64 reference itself
    # moves by up to ~2e-4 (normwise) when only its INPUTS are rounded at FP32 level
    # (6e-8).  Tolerance = max(1e-4, 20 x that measured sensitivity) normwise.
    sens = 0.0
    for k in range(3):
        r = np.random.default_rng(100 + k)
        fp_ = vpm.inject_ring(vpm.FluidState.empty(v), vpm.RingDisturbance.from_speed([0.8, -0.05], 7.5, 0.28,
                                                                                       0.02, -1.0))
        n = fp_.n_wake
        fp_.wake_pos[:n] *= 1.0 + 6e-8 * r.normal(size=(n, 2))
        d2 = oracle_core.batch_rollout_diag(X0 * (1.0 + 6e-8 * r.normal(size=7)), ctrl, *fp_.flat(), eng.iparams,
                                            eng.fparams, record=True)
        m = ok & (d2["status"] == 0)
        e = np.abs(d2["trajs"][m] - d["trajs"][m]).max(axis=(0, 1)) / np.abs(d["trajs"][m]).max(axis=(0, 1))
        sens = max(sens, float(e.max()))
    rtol = max(1e-4, 20.0 * sens)
    print(f"  nb={nb} cap={cap}: FP64 reference sensitivity to FP32-rounded inputs {sens:.2e} -> rtol {rtol:.2e}")
    TOL["edge"] = ("norm", rtol, 1e-9)
    assert_close(res.trajectories[ok], d["trajs"][ok], "edge", what="trajs")


def test_overfull_snapshot_and_reversed_flow(torch_cuda, oracle_core):
    """n_wake = cap + 4 at fork (overflow targets + 4-6 merges in one step) and a
    tail-first plate (|aoa| > 90 deg: reversed-flow rows and edge roles)."""
    from paper_2509_16079_b200 import config, rollout, vpm
    sc = golden("scenario_C3.npz")
    v = config.VpmConfig(particle_cap=128)  # register tile 64 x 2 = 128 < 132 particles
    eng = rollout.Engine(v, config.GliderParams())
    fl = vpm.FluidState.empty(v)
    keep = list(range(130)) + [int(sc["ring_a"]), int(sc["ring_b"])]
    n = len(keep)  # cap + 4
    fl.wake_pos[:n], fl.wake_gamma[:n], fl.wake_age[:n] = (sc["wake_pos"][keep], sc["wake_gamma"][keep],
                                                           sc["wake_age"][keep])
    fl.n_wake, fl.ring_a, fl.ring_b = n, 130, 131
    for x0 in (X0, np.array([0.0, 0.0, 0.2, 0.0, -6.0, 0.5, 0.0])):
        ctrl = np.full((3, 20), -4.0)
        ctrl[1] = 6.0
        ctrl[2] = np.linspace(-15, 15, 20)
        res = eng.batch(rollout.RolloutRequest(x0=x0, fluid=fl, controls=ctrl, record=True))
        d = oracle_core.batch_rollout_diag(x0, ctrl, *fl.flat(), eng.iparams, eng.fparams, record=True)
        np.testing.assert_array_equal(res.status, d["status"])
        ok = d["status"] == 0
        assert_close(res.trajectories[ok], d["trajs"][ok], what="trajs")


def test_envelope_blowup_status(torch_cuda, oracle_core):
    from paper_2509_16079_b200 import config, rollout, vpm
    v = config.VpmConfig(particle_cap=60)
    eng = rollout.Engine(v, config.GliderParams())
    fl = vpm.FluidState.empty(v)
    x0 = np.array([0.0, 0.0, 0.0, 0.0, 7.0, 0.0, 290.0])  # spins past |omega| > 300
    ctrl = np.full((2, 10), 15.0)
    res = eng.batch(rollout.RolloutRequest(x0=x0, fluid=fl, controls=ctrl))
    d = oracle_core.batch_rollout_diag(x0, ctrl, *fl.flat(), eng.iparams, eng.fparams)
    np.testing.assert_array_equal(res.status, d["status"])
    assert (res.status > 0).all()


def test_concurrent_callers_get_independent_results(torch_cuda):
    """The stepping module is called from two threads in threaded NMPC mode (plant
    loop + replanning worker, nmpc.py:219-222; SURVEY 8b 'Threading'): concurrent
    Engine.step / Engine.batch calls from several threads must return exactly what
    the same calls return one at a time."""
    import threading

    from paper_2509_16079_b200 import config, rollout, vpm
    cfg = config.ExperimentConfig()
    eng = rollout.Engine.from_config(cfg)
    x0 = np.array([0.0, 0.0, 0.3, 0.0, 7.0, 0.0, 0.0])

    def stepping(seed):
        fl, x = vpm.FluidState.empty(cfg.vpm), x0.copy()
        us = np.random.default_rng(seed).uniform(-15, 15, 40)
        out = []
        for u in us:
            ok, x, fl, _ = eng.step(x, u, fl)
            out.append(x.copy())
        return np.array(out), fl.wake_pos.copy()

    def batching(seed):
        u = np.random.default_rng(seed).uniform(-15, 15, (64, 30))
        res = eng.batch(rollout.RolloutRequest(x0=x0, fluid=vpm.FluidState.empty(cfg.vpm), controls=u))
        return res.status.copy(), res.finals.copy()

    jobs = [(stepping, s) for s in range(3)] + [(batching, s) for s in range(3)]
    serial = [fn(s) for fn, s in jobs]
    got = [None] * len(jobs)

    def run(i):
        for _ in range(3):
            got[i] = jobs[i][0](jobs[i][1])

    threads = [threading.Thread(target=run, args=(i,)) for i in range(len(jobs))]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    for a, b in zip(serial, got):
        for x, y in zip(a, b):
            np.testing.assert_array_equal(x, y)


def test_concurrent_optimize_on_one_engine(torch_cuda):
    """mppi.optimize / build_policy share the engine's device plan (snapshot and
    pinned staging); concurrent callers on one engine serialise on the plan's lock
    and get exactly their serial results."""
    import threading

    from paper_2509_16079_b200 import config, mppi, rollout, vpm
    cfg = config.ExperimentConfig()
    cfg.mppi.batch = 128
    eng = rollout.Engine.from_config(cfg)
    x0 = np.array([0.0, 0.0, 0.3, 0.0, 7.0, 0.0, 0.0])
    ring = vpm.RingDisturbance.from_speed([1.0, -0.1], 7.5, 0.28, 0.02, -1.0)
    fluids = [vpm.FluidState.empty(cfg.vpm), vpm.inject_ring(vpm.FluidState.empty(cfg.vpm), ring)]

    def job(i):
        rng = np.random.default_rng(40 + i)
        return mppi.optimize(x0, fluids[i % 2], np.full(cfg.mppi.horizon, -6.0), cfg.mppi, eng, rng,
                             iterations=2)

    serial = [job(i) for i in range(4)]
    got = [None] * 4

    def run(i):
        for _ in range(3):
            got[i] = job(i)

    threads = [threading.Thread(target=run, args=(i,)) for i in range(4)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    for a, b in zip(serial, got):
        np.testing.assert_array_equal(a, b)
    assert not np.array_equal(serial[0], serial[1])


def test_optimize_pipeline_equals_host_entry_and_rewinds_on_failure(torch_cuda):
    """mppi.optimize (per-iteration draws overlapped with the device) returns bitwise
    what the all-up-front C entry point vpm_mppi_optimize_host returns, and when
    every candidate fails it raises ValueError leaving the generator exactly where
    the reference leaves it (iteration 0's draw only)."""
    from paper_2509_16079_b200 import _lib, config, mppi
    from paper_2509_16079_b200._lib import _D, as_f64, ptr
    sc = golden("scenario_C2.npz")
    eng = engine_for(sc["iparams"], sc["fparams"])
    mcfg = config.MppiConfig(batch=256, iterations=3, horizon=50)
    fl = fluid_from(sc, 60)
    u_pipe = mppi.optimize(sc["x0"], fl, sc["warm"], mcfg, eng, np.random.default_rng(4))
    noise = as_f64(np.random.default_rng(4).normal(0.0, 1.0, (3, 256, 50)))
    plan = mppi.engine_plan(eng)
    plan.set_fluid(fl)
    u_host = np.clip(np.asarray(sc["warm"], float), -15, 15).copy()
    q, xp, x0 = as_f64(mcfg.q_terminal), as_f64(mcfg.x_perch), as_f64(sc["x0"])
    assert _lib.lib().vpm_mppi_optimize_host(plan.handle, ptr(x0, _D), ptr(u_host, _D), ptr(noise, _D), 3,
                                             256, 50, 2.0, 0.05, ptr(q, _D), ptr(xp, _D)) == 0
    np.testing.assert_array_equal(u_pipe, u_host)
    bad = np.asarray(sc["x0"], float).copy()
    bad[6] = 400.0  # leaves the envelope on the first step: every candidate fails
    rng, twin = np.random.default_rng(8), np.random.default_rng(8)
    with pytest.raises(ValueError):
        mppi.optimize(bad, fl, sc["warm"], mcfg, eng, rng)
    twin.normal(0.0, 1.0, (256, 50))
    assert rng.bit_generator.state == twin.bit_generator.state


@pytest.mark.parametrize("N", [1024, 2048])
def test_c5_large_wake_vs_oracle(torch_cuda, oracle_core, N):
    """C5-scale wakes (N = 1024 / 2048, random wake, attached flow so N
    stays fixed; symmetric-pair sweep on 8 / 16 tiles): a few rollouts of 5 steps
    against the FP64 oracle on identical inputs -- final states, and the wake the
    single-rollout path returns."""
    from paper_2509_16079_b200 import config, rollout, vpm
    rng = np.random.default_rng(N)
    v = config.VpmConfig(particle_cap=N)
    eng = rollout.Engine(v, config.GliderParams())
    fl = vpm.FluidState.empty(v)
    fl.wake_pos[:N] = rng.normal(0.0, 0.5, (N, 2)) - np.array([3.0, 0.0])
    fl.wake_gamma[:N] = rng.normal(0.0, 0.05, N)
    fl.n_wake = N
    x0 = np.array([0.0, 0.0, 0.0, 0.0, 7.0, 0.0, 0.0])
    ctrl = np.clip(rng.normal(0.0, 3.0, (4, 5)), -15, 15)
    res = eng.batch(rollout.RolloutRequest(x0=x0, fluid=fl, controls=ctrl, record=True))
    d = oracle_core.batch_rollout_diag(x0, ctrl, *fl.flat(), eng.iparams, eng.fparams, record=True)
    np.testing.assert_array_equal(res.status, d["status"])
    assert (res.status == 0).all()
    assert_close(res.trajectories, d["trajs"], what=f"C5 N={N} trajs")
    rc, _, fl_g = eng.rollout(x0, ctrl[0], fl)
    rc_o, _, flat_o = oracle_core.rollout(x0, ctrl[0], *fl.flat(), eng.iparams, eng.fparams, False, True)
    assert rc == rc_o == 0 and fl_g.n_wake == flat_o[3] == N
    np.testing.assert_array_equal(fl_g.wake_age[:N], flat_o[2][:N])
    assert_close(fl_g.wake_pos[:N], flat_o[0][:N], "wake_pos", what=f"C5 N={N} wake")


@pytest.mark.parametrize("cap,n0", [(400, 300), (300, 290), (640, 600), (512, 516), (1000, 900)])
def test_symmetric_tiles_vs_oracle(torch_cuda, oracle_core, cap, n0):
    """The symmetric-pair tile schedule at the edges of its tiling: partial and empty
    tiles (cap 400 / wake 300), odd tile counts (cap 300: 3 tiles, cap 640: 5),
    eight tiles with a partial last one (cap 1000), and an overfull snapshot
    (cap + 4 particles: the first step takes the direct fallback); shedding plate,
    wakes growing into the cap and merging.  Decisions (status, shed steps, final wake
    size, wake-index signature) exact off near-ties, trajectories within the stated
    tolerance, and every single-rollout call bitwise equal to its row of the batch
    (the tile count depends on the cap only)."""
    torch = torch_cuda
    from paper_2509_16079_b200 import config, rollout, vpm
    from paper_2509_16079_b200.device import DevicePlan
    rng = np.random.default_rng(cap + n0)
    v = config.VpmConfig(particle_cap=cap)
    eng = rollout.Engine(v, config.GliderParams())
    fl = vpm.FluidState.empty(v)
    fl.wake_pos[:n0] = rng.normal(0.0, 0.5, (n0, 2)) - np.array([3.0, 0.0])
    fl.wake_gamma[:n0] = rng.normal(0.0, 0.02, n0)
    fl.wake_age[:n0] = rng.integers(0, 400, n0)
    fl.n_wake = n0
    B, T = 6, 30
    ctrl = np.clip(-6.0 + 3.0 * rng.normal(0.0, 1.0, (B, T)), -15, 15)
    plan = DevicePlan(eng.iparams, eng.fparams)
    plan.set_fluid(fl.flat())
    dev = torch.device("cuda")
    out = plan.batch(torch.as_tensor(X0, device=dev), T, controls=torch.as_tensor(ctrl, device=dev), rows=B,
                     diagnostics=True)
    torch.cuda.synchronize()
    gpu = {k: t.cpu().numpy() for k, t in out.items()}
    # repeated launches are bitwise identical (a shared-memory race in the tile
    # schedule would show up as run-to-run differences)
    for _ in range(3):
        again = plan.batch(torch.as_tensor(X0, device=dev), T, controls=torch.as_tensor(ctrl, device=dev), rows=B,
                           diagnostics=True)
        torch.cuda.synchronize()
        for k, t in again.items():
            np.testing.assert_array_equal(t.cpu().numpy(), gpu[k])
    d = oracle_core.batch_rollout_diag(X0, ctrl, *fl.flat(), eng.iparams, eng.fparams, record=True)
    ok = _check_decisions(gpu, d, f"cap {cap}, wake {n0}")
    assert ok.sum() >= 3
    res = eng.batch(rollout.RolloutRequest(x0=X0, fluid=fl, controls=ctrl, record=True))
    np.testing.assert_array_equal(res.status, gpu["status"])
    np.testing.assert_array_equal(res.trajectories[:, -1][res.status == 0], gpu["finals"][res.status == 0])
    assert_close(res.trajectories[ok], d["trajs"][ok], what=f"cap {cap} wake {n0} trajs")
    for k in range(B):
        rc, traj, _ = eng.rollout(X0, ctrl[k], fl, record=True)
        assert rc == res.status[k]
        if rc == 0:
            np.testing.assert_array_equal(traj, res.trajectories[k])


@pytest.mark.parametrize("cap,n0", [(60, 40), (512, 500)])
def test_failure_time_wake_vs_oracle(torch_cuda, oracle_core, cap, n0):
    """A rollout that leaves the envelope mid-horizon returns the wake of its
    failure time (the reference's run_rollout semantics, _core.pyx:465-491): the
    direct sweep (cap 60) and the symmetric sweep (cap 512), whose advection has
    already rewritten the wake buffer when the control phase detects the failure, so
    the dump comes from the compacted copy."""
    from paper_2509_16079_b200 import config, rollout, vpm
    rng = np.random.default_rng(cap)
    v = config.VpmConfig(particle_cap=cap)
    eng = rollout.Engine(v, config.GliderParams())
    fl = vpm.FluidState.empty(v)
    fl.wake_pos[:n0] = rng.normal(0.0, 0.5, (n0, 2)) - np.array([3.0, 0.0])
    fl.wake_gamma[:n0] = rng.normal(0.0, 0.02, n0)
    fl.wake_age[:n0] = rng.integers(0, 300, n0)
    fl.n_wake = n0
    x0 = np.array([0.0, 0.0, 0.3, 0.0, 7.0, 30.0, 0.0])  # leaves the envelope after 3-7 steps
    ctrl = np.full(20, 15.0)
    rc, _, fl_g = eng.rollout(x0, ctrl, fl)
    rc_o, _, flat_o = oracle_core.rollout(x0, ctrl, *fl.flat(), eng.iparams, eng.fparams, False, True)
    assert rc == rc_o and 2 < rc < 20, (rc, rc_o)
    n = flat_o[3]
    assert fl_g.n_wake == n and (fl_g.ring_a, fl_g.ring_b) == (flat_o[4], flat_o[5])
    np.testing.assert_array_equal(fl_g.wake_age[:n], flat_o[2][:n])
    assert_close(fl_g.wake_pos[:n], flat_o[0][:n], "wake_pos", what=f"cap {cap} failure-time wake")
    assert_close(fl_g.wake_gamma[:n], flat_o[1][:n], "wake_gamma", what=f"cap {cap} failure-time gamma")
