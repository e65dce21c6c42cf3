"""Generate the golden fixtures in tests/golden/ from the REFERENCE itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports the unmodified reference package from /root/reference/pkg/src (numpy
backend = the readable FP64 specification, ``_accel/reference.py``) and records
its outputs on the synthetic perching scenarios of SURVEY.md section 8d.  The
fixtures are committed; nothing at test or bench time reads /root/reference.

Fixtures
  scenario_C2.npz  empty fluid, cap 60 (MPPI K=256, H=50)
  scenario_C3.npz  prefilled wake 254 + ring pair, cap 256 (K=1024)
  scenario_C4.npz  prefilled wake 510 + ring pair, cap 512 (K=4096)
  c1_steps.npz     C1 oracle rollout (empty fluid, cap 512, u=-15, 50 Engine.step calls)
  batch_ring.npz   32 rollouts on a prefilled 126-particle wake + ring, cap 128
  mppi_C2.npz      mppi.optimize, 3 iterations, C2 scenario, rng seed 0
  mppi_C3s.npz     one MPPI iteration with K=48 on the C3 scenario, rng seed 1
  policy_C2.npz    policy.build_policy around the C2 nominal, rng seed 2
  wake_sig.npz     (``make_golden.py wake_sig``) per-step shed / merge / ring
                   bookkeeping and final wake ages of MPPI candidate rollouts on the
                   C3 and C4 ring scenarios (H=50) and a C3 H=100 set, stepped with
                   the reference's Engine.step + the run_rollout envelope test
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = os.environ.get("REF_SRC", "/root/reference/pkg/src")
sys.path.insert(0, REF)
from perchsim import _accel, config, mppi, policy, rollout, vpm  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
H = 50
X0 = np.array([0.0, 0.0, 0.3, 0.0, 7.0, 0.0, 0.0])
RING_CENTER = (3.6, -0.1)


def flat(fl):
    return dict(wake_pos=fl.wake_pos.copy(), wake_gamma=fl.wake_gamma.copy(),
                wake_age=fl.wake_age.copy(), n_wake=fl.n_wake, ring_a=fl.ring_a,
                ring_b=fl.ring_b, prev_pos=fl.prev_pos.copy(), prev_gamma=fl.prev_gamma.copy(),
                n_prev=fl.n_prev, prev_lev=fl.prev_lev_gamma, ema=fl.unsteady_ema.copy())


def engine(cap):
    cfg = config.ExperimentConfig()
    cfg.vpm.particle_cap = cap
    return cfg, rollout.Engine(cfg.vpm, cfg.glider)


def prefilled(cap, n_target, ring=True):
    """plate held at theta=0.3 in a 7 m/s stream, stepped with
    fluid_step (x += 0.07 per step) until n_wake >= n_target, then translated so
    the plate sits at the head of its own wake; ring pair injected ahead."""
    cfg, eng = engine(cap)
    fl = vpm.FluidState.empty(cfg.vpm)
    x = X0.copy()
    while fl.n_wake < n_target:
        fl, _, _ = eng.fluid_step(x, fl)
        x[0] += 0.07
    fl.wake_pos[: fl.n_wake, 0] -= x[0]
    fl.prev_pos[: fl.n_prev, 0] -= x[0]
    if ring:
        fl = vpm.inject_ring(fl, vpm.RingDisturbance.from_speed(
            np.array(RING_CENTER), 7.5, 0.28, cfg.vpm.r_core, -1.0))
    return cfg, eng, fl


def save(name, **kw):
    np.savez_compressed(os.path.join(HERE, name), **kw)
    print("wrote", name, sum(np.asarray(v).nbytes for v in kw.values()), "bytes raw")


def main():
    assert _accel.active_backend() == "numpy", "expected the reference numpy backend"
    common = dict(x0=X0, warm=np.full(H, -6.0), stdev=2.0, temperature=0.05)

    # --- scenarios
    cfg2, eng2 = engine(60)
    fl2 = vpm.FluidState.empty(cfg2.vpm)
    save("scenario_C2.npz", cap=60, K=256, H=H, iparams=eng2.iparams, fparams=eng2.fparams,
         **flat(fl2), **common)
    cfg3, eng3, fl3 = prefilled(256, 254)
    save("scenario_C3.npz", cap=256, K=1024, H=H, iparams=eng3.iparams, fparams=eng3.fparams,
         **flat(fl3), **common)
    cfg4, eng4, fl4 = prefilled(512, 510)
    save("scenario_C4.npz", cap=512, K=4096, H=H, iparams=eng4.iparams, fparams=eng4.fparams,
         **flat(fl4), **common)

    # --- C1: 50 sequential Engine.step calls, u = -15, empty fluid, cap 512
    cfg1, eng1 = engine(512)
    fl = vpm.FluidState.empty(cfg1.vpm)
    x = X0.copy()
    xs, fws, ns, oks = [x.copy()], [], [], []
    for _ in range(H):
        ok, x, fl, fw = eng1.step(x, -15.0, fl)
        xs.append(x.copy()); fws.append(fw); ns.append(fl.n_wake); oks.append(ok)
    save("c1_steps.npz", iparams=eng1.iparams, fparams=eng1.fparams, states=np.array(xs),
         fw=np.array(fws), n_wake_steps=np.array(ns), ok=np.array(oks), **flat(fl))
    rc, traj, flr = eng1.rollout(X0, np.full(H, -15.0), vpm.FluidState.empty(cfg1.vpm), record=True)
    assert rc == 0 and np.array_equal(traj, np.array(xs)) and flr.n_wake == fl.n_wake

    # --- batch on a ring-disturbed prefilled wake
    cfgb, engb, flb = prefilled(128, 126)
    rng = np.random.default_rng(7)
    ctrl = np.clip(-6.0 + 3.0 * rng.normal(0.0, 1.0, (32, H)), -15, 15)
    res = engb.batch(rollout.RolloutRequest(x0=X0, fluid=flb, controls=ctrl, record=True))
    save("batch_ring.npz", iparams=engb.iparams, fparams=engb.fparams, controls=ctrl,
         status=res.status, finals=res.finals, trajs=res.trajectories, **flat(flb))

    # --- MPPI on C2 (3 iterations) with per-iteration costs captured
    class Tap(rollout.Engine):
        log = []

        def batch(self, req):
            r = super().batch(req)
            self.log.append((req.controls.copy(), r.status.copy(), r.finals.copy()))
            return r

    mcfg = config.MppiConfig(batch=256, iterations=3, horizon=H)
    tap = Tap(cfg2.vpm, cfg2.glider)
    u2 = mppi.optimize(X0, fl2, np.full(H, -6.0), mcfg, tap, np.random.default_rng(0))
    save("mppi_C2.npz", seed=0, K=256, iters=3, u_star=u2,
         costs=np.array([mppi.terminal_cost_batch(f, s, mcfg) for _, s, f in tap.log]),
         status=np.array([s for _, s, _ in tap.log]),
         finals=np.array([f for _, _, f in tap.log]),
         q=np.array(mcfg.q_terminal), x_perch=np.array(mcfg.x_perch))

    # --- one MPPI iteration, K=48, on the C3 ring scenario
    Tap.log = []
    mcfg3 = config.MppiConfig(batch=48, iterations=1, horizon=H)
    tap3 = Tap(cfg3.vpm, cfg3.glider)
    u3 = mppi.optimize(X0, fl3, np.full(H, -6.0), mcfg3, tap3, np.random.default_rng(1))
    c3, s3, f3 = tap3.log[0]
    save("mppi_C3s.npz", seed=1, K=48, iters=1, u_star=u3, status=s3, finals=f3,
         costs=mppi.terminal_cost_batch(f3, s3, mcfg3))

    # --- policy around the C2 nominal
    rc, traj, _ = eng2.rollout(X0, u2, fl2, record=True)
    assert rc == 0
    nom = policy.NominalTrajectory(states=traj, inputs=u2, dt=cfg2.vpm.dt)
    scfg = config.SynthesisConfig()
    pol = policy.build_policy(nom, fl2, scfg, eng2, np.random.default_rng(2))
    rng = np.random.default_rng(2)
    dx0 = rng.normal(0.0, 1.0, (scfg.n_samples, 7))
    du = rng.normal(0.0, 1.0, (scfg.n_samples, H))
    states, inputs, ok = policy.perturbed_rollouts(nom, fl2, scfg, eng2, np.random.default_rng(2))
    seq = policy.estimate_linear_sequence(nom, states, inputs, ok, cfg2.vpm.dt)
    save("policy_C2.npz", seed=2, nominal_states=traj, nominal_inputs=u2, gains=pol.gains,
         cloud_states=states, cloud_ok=ok, a_discrete=seq.a_discrete, b_discrete=seq.b_discrete,
         dx0=dx0, du=du)


def make_replan():
    """nmpc.bootstrap_policy (rng 0) then one nmpc.replan (rng 1) from x0 at t=0 with
    the default 10-step projection; default ExperimentConfig (cap 60, horizon 77,
    K=256).  Written to nmpc_replan.npz."""
    from perchsim import nmpc
    cfg = config.ExperimentConfig()
    eng = rollout.Engine.from_config(cfg)
    pol = nmpc.bootstrap_policy(cfg, eng, np.random.default_rng(0))
    fl0 = vpm.FluidState.empty(cfg.vpm)
    x0 = np.asarray(cfg.scenario.x0, dtype=float)
    proj = nmpc.project_forward(pol, x0, fl0, 0.0, cfg.scenario.t_proj_steps, eng)
    req = nmpc.ReplanRequest(x=x0, fluid=fl0, policy=pol, t=0.0, t_proj=cfg.scenario.t_proj_steps)
    new = nmpc.replan(req, cfg, eng, np.random.default_rng(1))
    assert proj is not None and new is not None
    xp, flp, tp = proj
    save("nmpc_replan.npz", boot_gains=pol.gains, boot_states=pol.nominal.states,
         boot_inputs=pol.nominal.inputs, proj_x=xp, proj_t=tp, proj_n_wake=flp.n_wake,
         proj_wake_pos=flp.wake_pos[: flp.n_wake], proj_wake_gamma=flp.wake_gamma[: flp.n_wake],
         proj_wake_age=flp.wake_age[: flp.n_wake], new_gains=new.gains,
         new_states=new.nominal.states, new_inputs=new.nominal.inputs, new_t_start=new.t_start)


def make_wake_sig():
    """Reference-side pin of the wake-index signature (tests/wake_sig.py): every
    rollout is stepped with the reference's Engine.step (numpy backend) and the
    run_rollout envelope / failure test (_core.pyx:465-491, reference.py:85-111);
    after each completed step the wake size, ring-core indices and the shed flag
    (a particle of age 0 exists: shed particles enter at age 0 after the step's
    ageing, _core.pyx:222-226, 322-334) are recorded, plus the final wake ages."""
    sys.path.insert(0, os.path.dirname(HERE))
    from wake_sig import signature
    out = {}
    for tag, name, K, H_, seed in (("c3", "scenario_C3.npz", 8, 50, 51), ("c4", "scenario_C4.npz", 8, 50, 52),
                                   ("c3long", "scenario_C3.npz", 4, 100, 53)):
        with np.load(os.path.join(HERE, name)) as z:
            sc = {k: z[k] for k in z.files}
        cap = int(sc["cap"])
        cfg, eng = engine(cap)
        fl0 = vpm.FluidState.empty(cfg.vpm)
        n0 = int(sc["n_wake"])
        fl0.wake_pos[:n0], fl0.wake_gamma[:n0], fl0.wake_age[:n0] = (sc["wake_pos"][:n0], sc["wake_gamma"][:n0],
                                                                     sc["wake_age"][:n0])
        fl0.n_wake, fl0.ring_a, fl0.ring_b = n0, int(sc["ring_a"]), int(sc["ring_b"])
        m = int(sc["n_prev"])
        fl0.prev_pos[:m], fl0.prev_gamma[:m], fl0.n_prev = sc["prev_pos"][:m], sc["prev_gamma"][:m], m
        fl0.prev_lev_gamma, fl0.unsteady_ema[:] = float(sc["prev_lev"]), sc["ema"]
        warm = np.full(H_, -6.0)
        noise = np.random.default_rng(seed).normal(0.0, 1.0, (K, H_))
        ctrl = np.clip(warm[None, :] + 2.0 * noise, -15.0, 15.0)
        status, sigs, nsteps, finals = [], [], [], []
        for k in range(K):
            fl, x, st, steps = fl0, X0.copy(), 0, []
            for t in range(H_):
                ok, x, fl, _ = eng.step(x, ctrl[k, t], fl)
                n = fl.n_wake
                steps.append((n, fl.ring_a, fl.ring_b, bool(np.any(fl.wake_age[:n] == 0))))
                if (not ok or not np.all(np.isfinite(x)) or abs(x[6]) > 300.0
                        or np.max(np.abs(x[4:6])) > 80.0):
                    st = 1 + t
                    break
            status.append(st)
            sigs.append(signature(steps, fl.wake_age[: fl.n_wake]))
            nsteps.append([s[0] for s in steps] + [-1] * (H_ - len(steps)))
            finals.append(x)
            print(tag, k, "status", st, "n", fl.n_wake, "shed steps", sum(s[3] for s in steps))
        out[tag + "_controls"] = ctrl
        out[tag + "_status"] = np.array(status, np.int64)
        out[tag + "_sig"] = np.array(sigs, np.uint64)
        out[tag + "_n_steps"] = np.array(nsteps, np.int64)
        out[tag + "_finals"] = np.array(finals)
    save("wake_sig.npz", **out)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "wake_sig":
        make_wake_sig()
        sys.exit(0)
    if len(sys.argv) > 1 and sys.argv[1] == "replan":
        make_replan()
        sys.exit(0)
    main()
