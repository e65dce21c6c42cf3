"""Pin the CPU oracle (oracle/vpm_oracle.c + oracle/planner.py) against golden
vectors produced by the reference itself (tests/golden/make_golden.py)."""
import numpy as np
import pytest

from conftest import flat_of, golden

X0 = np.array([0.0, 0.0, 0.3, 0.0, 7.0, 0.0, 0.0])
RTOL = 1e-9  # FP64 vs FP64, different accumulation order only


def test_c1_step_sequence_matches_reference(oracle_core):
    g = golden("c1_steps.npz")
    ip, fp = g["iparams"], g["fparams"]
    cap, nb = int(ip[1]), int(ip[0])
    fl = (np.zeros((cap + 4, 2)), np.zeros(cap + 4), np.zeros(cap + 4, np.int64), 0, -1, -1,
          np.zeros((nb, 2)), np.zeros(nb), 0, 0.0, np.zeros(nb))
    x = X0.copy()
    for t in range(50):
        rc, x, fw, mw, fl = oracle_core.step(x, -15.0, *fl, ip, fp, True)
        assert rc == 0
        assert fl[3] == g["n_wake_steps"][t]
        np.testing.assert_allclose(x, g["states"][t + 1], rtol=RTOL, atol=1e-11)
        np.testing.assert_allclose(fw, g["fw"][t], rtol=1e-8, atol=1e-10)
    n = int(g["n_wake"])
    assert fl[3] == n == 96
    np.testing.assert_allclose(fl[0][:n], g["wake_pos"][:n], rtol=RTOL, atol=1e-12)
    np.testing.assert_allclose(fl[1][:n], g["wake_gamma"][:n], rtol=1e-8, atol=1e-12)
    np.testing.assert_array_equal(fl[2][:n], g["wake_age"][:n])


def test_c1_rollout_equals_steps(oracle_core):
    g = golden("c1_steps.npz")
    ip, fp = g["iparams"], g["fparams"]
    cap, nb = int(ip[1]), int(ip[0])
    fl = (np.zeros((cap + 4, 2)), np.zeros(cap + 4), np.zeros(cap + 4, np.int64), 0, -1, -1,
          np.zeros((nb, 2)), np.zeros(nb), 0, 0.0, np.zeros(nb))
    rc, traj, flo = oracle_core.rollout(X0, np.full(50, -15.0), *fl, ip, fp, True, True)
    assert rc == 0 and flo[3] == 96
    np.testing.assert_allclose(traj, g["states"], rtol=RTOL, atol=1e-11)


def test_batch_ring_matches_reference(oracle_core):
    g = golden("batch_ring.npz")
    d = oracle_core.batch_rollout_diag(X0, g["controls"], *flat_of(g), g["iparams"], g["fparams"],
                                       record=True)
    np.testing.assert_array_equal(d["status"], g["status"])
    np.testing.assert_allclose(d["trajs"], g["trajs"], rtol=1e-8, atol=1e-10)


def test_batch_workers_bit_identical(oracle_core):
    g = golden("batch_ring.npz")
    a = oracle_core.batch_rollout_diag(X0, g["controls"][:8], *flat_of(g), g["iparams"],
                                       g["fparams"], record=True, workers=1)
    b = oracle_core.batch_rollout_diag(X0, g["controls"][:8], *flat_of(g), g["iparams"],
                                       g["fparams"], record=True, workers=4)
    assert np.array_equal(a["trajs"], b["trajs"]) and np.array_equal(a["status"], b["status"])


def test_mppi_C2_matches_reference(oracle_core):
    from oracle import planner
    g = golden("mppi_C2.npz")
    sc = golden("scenario_C2.npz")
    K, H = int(g["K"]), 50
    noise = np.random.default_rng(int(g["seed"])).normal(0.0, 1.0, (int(g["iters"]), K, H))
    trace = []
    u = planner.optimize(sc["x0"], flat_of(sc), sc["warm"], noise, sc["iparams"], sc["fparams"],
                         stdev=float(sc["stdev"]), temperature=float(sc["temperature"]),
                         q=g["q"], x_perch=g["x_perch"], u_limit=15.0, trace=trace)
    for it, tr in enumerate(trace):
        np.testing.assert_array_equal(tr["status"], g["status"][it])
        fin = np.isfinite(g["costs"][it])
        assert np.array_equal(np.isfinite(tr["costs"]), fin)
        np.testing.assert_allclose(tr["costs"][fin], g["costs"][it][fin], rtol=1e-8)
    np.testing.assert_allclose(u, g["u_star"], rtol=1e-7, atol=1e-9)


def test_mppi_C3_ring_iteration_matches_reference(oracle_core):
    from oracle import planner
    g = golden("mppi_C3s.npz")
    sc = golden("scenario_C3.npz")
    noise = np.random.default_rng(int(g["seed"])).normal(0.0, 1.0, (1, int(g["K"]), 50))
    trace = []
    u = planner.optimize(sc["x0"], flat_of(sc), sc["warm"], noise, sc["iparams"], sc["fparams"],
                         stdev=2.0, temperature=0.05, q=[10, 10, 1, 0, 0.2, 0.2, 0.2],
                         x_perch=[3.5, 0, np.pi / 4, 0, 0.5, -0.5, 0], u_limit=15.0, trace=trace)
    np.testing.assert_array_equal(trace[0]["status"], g["status"])
    np.testing.assert_allclose(trace[0]["finals"], g["finals"], rtol=1e-8, atol=1e-10)
    np.testing.assert_allclose(u, g["u_star"], rtol=1e-7, atol=1e-9)


def test_policy_C2_matches_reference(oracle_core):
    from oracle import planner
    g = golden("policy_C2.npz")
    sc = golden("scenario_C2.npz")
    states, U, ok = planner.perturbed_cloud(
        g["nominal_states"], g["nominal_inputs"], flat_of(sc), sc["iparams"], sc["fparams"],
        g["dx0"], g["du"], [1e-3, 1e-3, 5e-3, 5e-3, 0.05, 0.05, 0.05], 0.5, 15.0)
    np.testing.assert_array_equal(ok, g["cloud_ok"])
    np.testing.assert_allclose(states[ok], g["cloud_states"][ok], rtol=1e-8, atol=1e-10)
    Ad, Bd = planner.fit_sequence(g["nominal_states"], g["nominal_inputs"], states, U, ok, 0.01)
    np.testing.assert_allclose(Ad, g["a_discrete"], rtol=1e-5, atol=1e-8)
    np.testing.assert_allclose(Bd, g["b_discrete"], rtol=1e-5, atol=1e-8)
    K = planner.riccati_gains(Ad, Bd, [0.1, 0.1, 5.0, 0.1, 0.1, 0.1, 5.0], 0.01,
                              [400.0, 400.0, 10.0, 1.0, 1.0, 1.0, 1.0])
    np.testing.assert_allclose(K, g["gains"], rtol=1e-5, atol=1e-6)


def test_refcore_agrees_with_oracle_when_built(oracle_core):
    from oracle import refcore
    ref = refcore.load()
    if ref is None:
        pytest.skip("oracle/_ref not built")
    g = golden("batch_ring.npz")
    s, f, t = ref.batch_rollout(X0, np.ascontiguousarray(g["controls"][:8]), *flat_of(g),
                                g["iparams"], g["fparams"], True, 2)
    d = oracle_core.batch_rollout_diag(X0, g["controls"][:8], *flat_of(g), g["iparams"],
                                       g["fparams"], record=True)
    np.testing.assert_array_equal(s, d["status"])
    np.testing.assert_allclose(t, d["trajs"], rtol=1e-9, atol=1e-11)


@pytest.mark.parametrize("tag,name", [("c3", "scenario_C3.npz"), ("c4", "scenario_C4.npz"),
                                      ("c3long", "scenario_C3.npz")])
def test_wake_signature_matches_reference(oracle_core, tag, name):
    """The oracle's wake-index signature (per-step wake size / ring indices / shed
    flag chain + final index->age sum) equals the one computed from the reference's
    own Engine.step sequence (tests/golden/make_golden.py wake_sig), on MPPI
    candidates of the C3 / C4 ring scenarios (merging at cap every shed step) and on
    H=100 rollouts (shed bits past step 64); per-step wake sizes and the shed
    bitmask agree with it."""
    g = golden("wake_sig.npz")
    sc = golden(name)
    ctrl = g[tag + "_controls"]
    d = oracle_core.batch_rollout_diag(sc["x0"], ctrl, *flat_of(sc), sc["iparams"], sc["fparams"],
                                       per_step_n=True)
    np.testing.assert_array_equal(d["status"], g[tag + "_status"])
    np.testing.assert_array_equal(d["wake_hash"], g[tag + "_sig"])
    ns = g[tag + "_n_steps"]
    np.testing.assert_array_equal(np.where(ns >= 0, d["n_steps"], -1), ns)
    np.testing.assert_allclose(d["finals"], g[tag + "_finals"], rtol=1e-9, atol=1e-11)
    T = ctrl.shape[1]
    bits = [(int(d["shed_mask"][k]) | (int(d["shed_mask_hi"][k]) << 64)) for k in range(len(ctrl))]
    assert any(b >> 64 for b in bits) or T <= 64
    assert all(b < (1 << T) for b in bits)


def test_wake_signature_sensitive_to_order(oracle_core):
    """The signature is a real check: it changes when two final ages swap places
    or a step's merge count moves to another step."""
    import sys, os
    sys.path.insert(0, os.path.dirname(__file__))
    from wake_sig import signature
    steps = [(10, -1, -1, True), (10, -1, -1, False)]
    a = signature(steps, [3, 2, 1])
    assert a != signature(steps, [2, 3, 1])
    assert a != signature([(12, -1, -1, True), (10, -1, -1, False)], [3, 2, 1])
    assert a != signature([(10, 4, 5, True), (10, -1, -1, False)], [3, 2, 1])
