"""NMPC executive and experiment harness (reference
perchsim/nmpc.py and SPEC.md experiment-cli / acceptance criteria 1, 4, 8, 10).

CPU tests cover the host logic (SPSC worker contract with a stand-in replan, CLI
config handling, perch-error metric).  GPU tests run the executive on the device:
the sensor's induced-velocity kernel against a brute-force FP64 sum, ring
self-advection, deterministic trials, mode equivalence, observed-wake fidelity,
threaded mode, 30 trials against the reference executive's own outcomes
(tests/golden/ref_trials.json), and the initial-condition sweep.
"""
import dataclasses
import json
import math
import os

import numpy as np
import pytest

from paper_2509_16079_b200 import cli, nmpc
from paper_2509_16079_b200.config import ExperimentConfig
from paper_2509_16079_b200.replan import ReplanRequest


# ------------------------------------------------------------------------ CPU: host logic
class _FakeEngine:
    class cfg:  # noqa: N801 - mirrors Engine.cfg
        dt = 0.01


def _request(t, t_proj=10):
    return ReplanRequest(x=np.zeros(7), fluid=None, policy=None, t=t, t_proj=t_proj)


@pytest.mark.parametrize("threaded", [False, True])
def test_worker_spsc_contract(monkeypatch, threaded):
    """One outstanding request; result released only at t_new and once finished
    (nmpc.py:191-238)."""
    calls = []

    def fake_replan(req, cfg, engine, rng):
        calls.append(req.t)
        return ("policy", req.t)

    monkeypatch.setattr(nmpc, "replan", fake_replan)
    w = nmpc._WorkerHandle(None, _FakeEngine(), None, threaded=threaded)
    assert w.poll(0.0) == (None, False)  # nothing outstanding
    w.request(_request(0.0))
    with pytest.raises(RuntimeError):
        w.request(_request(0.0))  # single outstanding request
    w.join()
    assert w.poll(0.05) == (None, False)  # budget not elapsed
    assert w.status == w.BUSY
    pol, done = w.poll(0.1)  # t_new = 0 + 10 * 0.01
    assert done and pol == ("policy", 0.0)
    assert w.status == w.READY and calls == [0.0]
    assert w.poll(1.0) == (None, False)


def test_worker_rejected_replan_is_reported(monkeypatch):
    monkeypatch.setattr(nmpc, "replan", lambda *a: None)
    w = nmpc._WorkerHandle(None, _FakeEngine(), None, threaded=False)
    w.request(_request(0.3, t_proj=0))
    assert w.poll(0.3) == (None, True)


def test_worker_failure_is_raised_not_a_stale_policy(monkeypatch):
    """A replan that raises in the threaded worker must surface from poll(), never
    hand back the previous cycle's policy as a fresh replan."""
    results = iter([("policy", 0.0)])

    def flaky(req, cfg, engine, rng):
        try:
            return next(results)
        except StopIteration:
            raise FloatingPointError("device failure") from None

    monkeypatch.setattr(nmpc, "replan", flaky)
    w = nmpc._WorkerHandle(None, _FakeEngine(), None, threaded=True)
    w.request(_request(0.0))
    w.join()
    assert w.poll(0.1) == (("policy", 0.0), True)
    w.request(_request(0.1))
    w.join()
    with pytest.raises(RuntimeError, match="replanning worker failed"):
        w.poll(0.2)
    assert w.status == w.READY


def test_pressure_trigger_empty_wake_never_fires():
    from paper_2509_16079_b200.vpm import FluidState
    fl = FluidState.empty(ExperimentConfig().vpm)
    assert not nmpc.pressure_trigger([3.4, -0.35], fl, 1.2, 0.02, 15.0)
    assert nmpc.pressure_trigger([3.4, -0.35], fl, 1.2, 0.02, 0.0)  # 0 >= 0, no device call


def test_estimated_ring_is_anchored_at_the_sensor():
    cfg = ExperimentConfig()
    true_ring, est = nmpc._true_ring(cfg), nmpc._estimated_ring(cfg)
    assert est.center[0] == cfg.scenario.sensor_pos[0]
    assert est.center[1] == cfg.scenario.ring_center[1] + cfg.scenario.est_height_offset
    assert math.isclose(est.circulation, true_ring.circulation, rel_tol=1e-15)
    sc = dataclasses.replace(cfg.scenario, est_circulation_scale=1.5, est_separation_scale=0.5)
    est2 = nmpc._estimated_ring(dataclasses.replace(cfg, scenario=sc))
    assert est2.separation == 0.5 * cfg.scenario.ring_separation


def test_perch_error_metric_first_crossing():
    traj = np.zeros((5, 7))
    traj[:, 0] = [0.0, 1.0, 3.6, 3.9, 4.0]
    traj[:, 1] = [0.0, 0.0, 0.3, 0.5, 0.6]
    assert math.isclose(cli._perch_error(traj, (3.5, 0.0)), math.hypot(0.1, 0.3))
    traj[:, 0] = [0.0, 1.0, 2.0, 3.0, 3.4]
    assert math.isclose(cli._perch_error(traj, (3.5, 0.0)), math.hypot(0.1, 0.6))


def test_cli_validate_config(tmp_path, capsys):
    good = tmp_path / "good.json"
    good.write_text(json.dumps({"trials": 2, "scenario": {"mode": "compensated"}}))
    assert cli.main(["validate-config", "--config", str(good)]) == 0
    assert json.loads(capsys.readouterr().out)["valid"]
    bad = tmp_path / "bad.json"
    bad.write_text(json.dumps({"scenario": {"nope": 1}}))
    assert cli.main(["validate-config", "--config", str(bad)]) == 2
    assert "scenario.nope" in capsys.readouterr().err


def test_trial_csv_layout(tmp_path):
    rec = nmpc.TrialRecord(seed=3, mode="compensated", dt=0.01, times=np.array([0.0, 0.01]),
                           states=np.arange(14.0).reshape(2, 7), inputs=np.array([1.0, -2.0]),
                           wake_counts=np.array([0, 2]), replanned=np.array([0, 1]))
    p = tmp_path / "t.csv"
    cli.write_trial_csv(rec, str(p), "abc")
    lines = p.read_text().splitlines()
    assert lines[0].startswith("# config_hash=abc mode=compensated seed=3")
    assert lines[1].split(",") == list(cli.CSV_COLUMNS)
    assert lines[3].split(",")[-3:] == ["-2.0", "2", "1"]


# ------------------------------------------------------------------------ GPU
def _small_cfg(**scenario):
    cfg = ExperimentConfig()
    return dataclasses.replace(cfg, scenario=dataclasses.replace(cfg.scenario, **scenario))


@pytest.mark.gpu
def test_induced_velocity_matches_bruteforce_and_kernel_limits():
    """SPEC acceptance 1: summation vs a brute-force pairwise FP64 oracle to 1e-12;
    regularised within 1% of singular for r >= 5 r_core; zero self-velocity."""
    from paper_2509_16079_b200.vpm import induced_velocity, induced_velocity_at
    rng = np.random.default_rng(7)
    pos, gam = rng.normal(0, 0.5, (50, 2)), rng.normal(0, 0.05, 50)
    tg = rng.normal(0, 0.5, (9, 2))
    rc = 0.02
    got = induced_velocity_at(tg, pos, gam, r_core=rc)
    ref = np.zeros_like(tg)
    for i, t in enumerate(tg):
        for p, g in zip(pos, gam):
            dx, dz = t - p
            c = g / (2 * math.pi * math.sqrt((dx * dx + dz * dz) ** 2 + rc ** 4))
            ref[i] += (c * dz, -c * dx)
    np.testing.assert_allclose(got, ref, rtol=1e-12, atol=1e-15)
    one = np.array([[0.0, 0.0]])
    for r in (5 * rc, 10 * rc, 1.0):
        reg = induced_velocity(one, [1.0], [r, 0.0], r_core=rc)
        sing = induced_velocity(one, [1.0], [r, 0.0], kernel="singular")
        assert abs(reg[1] - sing[1]) <= 0.01 * abs(sing[1])
    assert np.all(induced_velocity(one, [1.0], [0.0, 0.0], r_core=rc) == 0.0)
    assert np.all(induced_velocity(one, [1.0], [0.0, 0.0], kernel="singular") == 0.0)
    with pytest.raises(ValueError):
        induced_velocity(one, [1.0], [1.0, 0.0], kernel="bogus")


@pytest.mark.gpu
def test_ring_self_advects_at_design_speed():
    """SPEC acceptance 4: a ring pair built for 7.5 m/s, d = 0.28, translates at
    7.5 m/s +-5% over 50 steps with dissipation off (plate parked far away)."""
    from paper_2509_16079_b200.rollout import Engine
    from paper_2509_16079_b200.vpm import FluidState, RingDisturbance, inject_ring
    cfg = ExperimentConfig()
    cfg = dataclasses.replace(cfg, vpm=dataclasses.replace(cfg.vpm, k_dissipation=1.0))
    eng = Engine.from_config(cfg)
    fl = inject_ring(FluidState.empty(cfg.vpm),
                     RingDisturbance.from_speed([0.0, 0.0], 7.5, 0.28, cfg.vpm.r_core, direction=1.0))
    x_far = np.array([500.0, 500.0, 0.0, 0.0, 0.0, 0.0, 0.0])
    c0 = fl.wake_pos[:2].mean(axis=0)
    for _ in range(50):
        fl, _, _ = eng.fluid_step(x_far, fl)
    assert fl.n_wake == 2
    c1 = fl.wake_pos[:2].mean(axis=0)
    speed = float(np.hypot(*(c1 - c0))) / (50 * cfg.vpm.dt)
    assert abs(speed - 7.5) <= 0.05 * 7.5
    assert c1[0] > c0[0]  # direction +1 travels along +x


@pytest.mark.gpu
def test_trial_is_deterministic_and_modes_agree_without_ring():
    """SPEC acceptance 10 + 'deterministic per seed': simulated-time trials are a
    function of (config, mode, seed); with no ring fired all modes coincide."""
    cfg = _small_cfg(fire_step=-1, max_steps=60)
    recs = {m: nmpc.control_loop(cfg, m, 4) for m in nmpc.MODES}
    again = nmpc.control_loop(cfg, nmpc.MODE_COMPENSATED, 4)
    base = recs[nmpc.MODE_NO_DISTURBANCE]
    assert len(base.times) > 10 and base.failure is None
    assert any(e.accepted for e in base.replans)
    for r in (*recs.values(), again):
        np.testing.assert_array_equal(r.states, base.states)
        np.testing.assert_array_equal(r.inputs, base.inputs)
        np.testing.assert_array_equal(r.replanned, base.replanned)
    # adoption happens exactly t_proj ticks after each request
    for ev in base.replans:
        if ev.accepted:
            assert math.isclose(ev.t_new - ev.t_request, cfg.scenario.t_proj_steps * cfg.vpm.dt, abs_tol=1e-9)
            assert ev.projection_gap < 0.05


@pytest.mark.gpu
def test_observed_wake_tracks_truth_without_disturbance():
    """SPEC invariant 'observed-wake fidelity': with a perfect model and no ring the
    observed wake equals the plant-truth wake step for step."""
    from paper_2509_16079_b200.rollout import Engine
    from paper_2509_16079_b200.vpm import FluidState
    cfg = ExperimentConfig()
    eng = Engine.from_config(cfg)
    x = np.array([0.0, 0.0, 0.3, 0.0, 7.0, 0.0, 0.0])  # pitched up: sheds from the first step
    truth, obs = FluidState.empty(cfg.vpm), FluidState.empty(cfg.vpm)
    for k in range(30):
        u = -6.0 + 0.2 * k
        x_prev = x.copy()
        ok, x, truth, _ = eng.step(x, u, truth)
        obs, _, _ = eng.fluid_step(x_prev, obs)
        assert ok and truth.equals(obs)
    assert truth.n_wake > 0


@pytest.mark.gpu
def test_threaded_mode_runs_and_adopts():
    cfg = _small_cfg(loop_mode="threaded", max_steps=80)
    rec = nmpc.control_loop(cfg, nmpc.MODE_UNCOMPENSATED, 1)
    assert len(rec.times) > 20
    assert sum(e.accepted for e in rec.replans) >= 1
    assert np.isfinite(rec.final_error)


@pytest.mark.gpu
def test_ring_trigger_and_compensated_injection():
    cfg = _small_cfg()
    rec = nmpc.control_loop(cfg, nmpc.MODE_COMPENSATED, 0)
    assert rec.trigger_time is not None
    assert rec.trigger_time >= cfg.scenario.fire_step * cfg.vpm.dt - 1e-9
    # threshold = infinity: compensated degenerates to uncompensated
    inf = _small_cfg(trigger_threshold_pa=math.inf)
    a = nmpc.control_loop(inf, nmpc.MODE_COMPENSATED, 0)
    b = nmpc.control_loop(inf, nmpc.MODE_UNCOMPENSATED, 0)
    assert a.trigger_time is None
    np.testing.assert_array_equal(a.states, b.states)


@pytest.mark.gpu
def test_cli_trial_outputs_are_reproducible(tmp_path):
    out1, out2 = tmp_path / "a", tmp_path / "b"
    args = ["trial", "--mode", "no_disturbance", "--trials", "1", "--seed", "2"]
    assert cli.main(args + ["--out", str(out1)]) == 0
    assert cli.main(args + ["--out", str(out2)]) == 0
    for name in os.listdir(out1):
        assert (out1 / name).read_bytes() == (out2 / name).read_bytes()
    summ = json.loads((out1 / "summary.json").read_text())
    assert summ["schema"] == cli.SCHEMA and summ["modes"]["no_disturbance"]["trials"] == 1


@pytest.mark.gpu
def test_trials_reproduce_the_reference_executive():
    """30 closed-loop trials (3 modes x seeds 0-9, ExperimentConfig defaults) against
    the unmodified reference executive run on its own compiled FP64 core
    (tests/golden/ref_trials.json, made by tools/ref_trials.py).  Every trial must
    end at the same tick with the same replan count and its final perch error within
    1e-4 m; the medians then reproduce the reference's ordering
    no_disturbance <= compensated < uncompensated (SPEC acceptance 8).  The SPEC's
    extra 60% margin is not met by the reference itself (0.451 / 0.559 = 0.81), so
    it is reported, not asserted."""
    with open(os.path.join(os.path.dirname(__file__), "golden", "ref_trials.json")) as fh:
        ref = json.load(fh)["trials"]
    summary, recs = cli.run_trials(ExperimentConfig(), nmpc.MODES, 10, seed_base=0)
    worst = 0.0
    for mode, rs in recs.items():
        for r in rs:
            g = ref[f"{mode}/{r.seed}"]
            assert len(r.times) == g["steps"], (mode, r.seed)
            assert sum(e.accepted for e in r.replans) == g["replans_accepted"], (mode, r.seed)
            assert (r.failure is None) == (g["failure"] is None)
            worst = max(worst, abs(r.final_error - g["final_error"]))
    med = {k: summary["modes"][k]["median_error_m"] for k in nmpc.MODES}
    print(json.dumps({"medians": med, "worst_final_error_diff_m": worst}))
    assert worst <= 1e-4
    assert med[nmpc.MODE_NO_DISTURBANCE] <= med[nmpc.MODE_COMPENSATED] < med[nmpc.MODE_UNCOMPENSATED]


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["no_disturbance", "uncompensated", "compensated"])
def test_resident_loop_equals_host_stepping(mode):
    """The control loop with both fluids kept on the device (vpm_plan_step in place,
    one sync per tick) is bitwise the loop that steps through the reference's
    host-buffer contract (Engine.step / fluid_step every tick)."""
    cfg = ExperimentConfig()
    a = nmpc.control_loop(cfg, mode, 3, resident=True)
    b = nmpc.control_loop(cfg, mode, 3, resident=False)
    np.testing.assert_array_equal(a.states, b.states)
    np.testing.assert_array_equal(a.inputs, b.inputs)
    np.testing.assert_array_equal(a.wake_counts, b.wake_counts)
    assert a.trigger_time == b.trigger_time and a.failure == b.failure
    assert [e.accepted for e in a.replans] == [e.accepted for e in b.replans]


@pytest.mark.gpu
def test_initial_condition_sweep():
    """SPEC run_sweep (Fig. 'ic-sweep'): v_x swept about the nominal 7 m/s; the
    nominal point is included; TVLQR feedback is reported beside the open loop."""
    res = cli.run_sweep(ExperimentConfig(), 5, -0.3, 0.3, 7, seed=0)
    rows = res["rows"]
    print(json.dumps(rows))
    assert len(rows) == 7 and any(abs(r["delta"]) < 1e-12 for r in rows)
    assert all(math.isfinite(r["closed_loop_error_m"]) for r in rows)
    mid = [r for r in rows if abs(r["delta"]) < 1e-12][0]
    assert mid["x0_value"] == 7.0
