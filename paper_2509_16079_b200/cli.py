"""Experiment harness (SPEC.md experiment-cli: ``trial``, ``sweep``, ``bench``,
``validate-config``; declared by the reference's pyproject, absent from its tree).

    python -m paper_2509_16079_b200 trial  [--config C] [--mode M|all] [--trials N] [--seed S] [--out DIR]
    python -m paper_2509_16079_b200 sweep  [--config C] [--state 5] [--lo -0.3] [--hi 0.3] [--steps 7]
    python -m paper_2509_16079_b200 bench  [--config C] [--batches 1,128,256,512,1024] [--horizon 80]
    python -m paper_2509_16079_b200 validate-config --config C

Outputs: one CSV per trial (columns ``t, r_x, r_z, theta, phi, v_x, v_z, omega, u,
wake_count, replanned``; a leading comment line carries the config hash, mode and
seed) and a versioned JSON summary; ``sweep`` and ``bench`` print one JSON document
and write a CSV when ``--out`` is given.  Every run embeds the config hash; identical
(config, seed) gives identical files.  Exit code 0 only when every requested run
completed.
"""

from __future__ import annotations

import argparse
import dataclasses
import json
import os
import sys
import time

import numpy as np

from . import config as config_mod
from .config import ConfigError, ExperimentConfig
from .nmpc import MODES, TrialRecord, bootstrap_policy, control_loop
from .policy import evaluate_policy
from .rollout import Engine, RolloutRequest
from .vpm import FluidState

SCHEMA = 1
CSV_COLUMNS = ("t", "r_x", "r_z", "theta", "phi", "v_x", "v_z", "omega", "u", "wake_count", "replanned")
STATE_NAMES = ("r_x", "r_z", "theta", "phi", "v_x", "v_z", "omega")


def _quartiles(values) -> dict:
    v = np.asarray(values, dtype=float)
    if v.size == 0:
        return {"median_error_m": None, "q25": None, "q75": None}
    q25, med, q75 = np.percentile(v, [25, 50, 75])
    return {"median_error_m": float(med), "q25": float(q25), "q75": float(q75)}


def write_trial_csv(rec: TrialRecord, path: str, cfg_hash: str) -> None:
    with open(path, "w") as fh:
        fh.write(f"# config_hash={cfg_hash} mode={rec.mode} seed={rec.seed} schema={SCHEMA}\n")
        fh.write(",".join(CSV_COLUMNS) + "\n")
        for i in range(len(rec.times)):
            s = rec.states[i]
            row = [rec.times[i], *s, rec.inputs[i]]
            fh.write(",".join(repr(float(v)) for v in row))
            fh.write(f",{int(rec.wake_counts[i])},{int(rec.replanned[i])}\n")


def run_trials(cfg: ExperimentConfig, modes, n_trials: int, seed_base: int | None = None,
               out_dir: str | None = None):
    """``n_trials`` paired seeds per mode (SPEC run_trials); returns (summary, records)."""
    base = cfg.seed_base if seed_base is None else seed_base
    h = cfg.config_hash()
    records = {}
    summary = {"schema": SCHEMA, "config_hash": h, "seed_base": base, "trials": n_trials, "modes": {}}
    if out_dir:
        os.makedirs(out_dir, exist_ok=True)
    for mode in modes:
        recs = []
        for i in range(n_trials):
            c = dataclasses.replace(cfg, scenario=dataclasses.replace(cfg.scenario, mode=mode))
            rec = control_loop(c, mode, base + i)
            recs.append(rec)
            if out_dir:
                write_trial_csv(rec, os.path.join(out_dir, f"trial_{mode}_seed{base + i}.csv"), h)
        records[mode] = recs
        errs = [r.final_error for r in recs]
        summary["modes"][mode] = {**_quartiles(errs), "trials": len(recs),
                                  "failures": sum(r.failure is not None for r in recs),
                                  "errors_m": [float(e) for e in errs],
                                  "replans_accepted": sum(sum(e.accepted for e in r.replans) for r in recs)}
    m = summary["modes"]
    if all(k in m for k in MODES):
        nd, co, un = (m[k]["median_error_m"] for k in MODES)
        summary["ordering"] = {"no_disturbance<=compensated<uncompensated": bool(nd <= co < un),
                               "compensated_over_uncompensated": co / un if un else None}
    if out_dir:
        with open(os.path.join(out_dir, "summary.json"), "w") as fh:
            json.dump(summary, fh, indent=1, sort_keys=True)
    return summary, records


def _perch_error(traj: np.ndarray, perch_xy) -> float:
    """Distance to the perch point when r_x first crosses the perch plane, else at the
    end of the trajectory (SPEC design decision 'perch-error metric')."""
    hit = np.nonzero(traj[:, 0] >= perch_xy[0])[0]
    s = traj[hit[0]] if hit.size else traj[-1]
    return float(np.hypot(s[0] - perch_xy[0], s[1] - perch_xy[1]))


def _terminal_cost(x, cfg: ExperimentConfig) -> float:
    d = np.asarray(x, float) - np.asarray(cfg.mppi.x_perch, float)
    return float(np.sum(np.asarray(cfg.mppi.q_terminal, float) * d * d))


def run_sweep(cfg: ExperimentConfig, state: int, lo: float, hi: float, steps: int, seed: int | None = None):
    """Initial-condition sweep (SPEC run_sweep, Fig. 'ic-sweep'): perturb state
    ``state`` (1-based) of x0 over [lo, hi]; for each point fly the bootstrap plan
    open loop and under its TVLQR policy (no replanning), and report final costs and
    perch errors."""
    if not 1 <= state <= 7:
        raise ValueError("state index must be in 1..7")
    seed = cfg.seed_base if seed is None else seed
    engine = Engine.from_config(cfg)
    rng = np.random.default_rng(seed)
    policy = bootstrap_policy(cfg, engine, rng)
    nom = policy.nominal
    perch = np.asarray(cfg.mppi.x_perch[:2], float)
    u_lim = engine.params.u_limit
    x_nom = np.asarray(cfg.scenario.x0, float)
    rows = []
    for delta in np.linspace(lo, hi, steps) if steps > 1 else [lo]:
        x0 = x_nom.copy()
        x0[state - 1] += delta
        # open loop: the nominal inputs from the perturbed start
        rc, traj, _ = engine.rollout(x0, nom.inputs, FluidState.empty(cfg.vpm), record=True)
        n_ok = len(traj) if rc == 0 else int(rc)
        ol = traj[:max(n_ok, 1)]
        # closed loop: TVLQR feedback around the nominal, plant stepped tick by tick
        x, fl, t = x0.copy(), FluidState.empty(cfg.vpm), nom.t_start
        cl = [x.copy()]
        ok = True
        for _ in range(nom.horizon):
            u = evaluate_policy(policy, x, t, u_lim)
            ok, x, fl, _ = engine.step(x, u, fl)
            t += nom.dt
            if not ok:
                break
            cl.append(x.copy())
            if x[0] >= perch[0]:
                break
        cl = np.asarray(cl)
        rows.append({"delta": float(delta), "x0_value": float(x0[state - 1]),
                     "open_loop_cost": _terminal_cost(ol[-1], cfg) if rc == 0 else float("inf"),
                     "closed_loop_cost": _terminal_cost(cl[-1], cfg) if ok else float("inf"),
                     "open_loop_error_m": _perch_error(ol, perch),
                     "closed_loop_error_m": _perch_error(cl, perch),
                     "open_loop_status": int(rc), "closed_loop_ok": bool(ok)})
    return {"schema": SCHEMA, "config_hash": cfg.config_hash(), "seed": seed, "state": STATE_NAMES[state - 1],
            "rows": rows}


def run_bench(cfg: ExperimentConfig, batches=(1, 128, 256, 512, 1024), horizon: int = 80, cap: int = 60,
              repeats: int = 5, seed: int = 0):
    """Batch-runtime table (SPEC run_bench): ``horizon``-step
    rollouts from x0 = [0,0,0.3,0,7,0,0] on an empty wake with particle cap ``cap``,
    controls clip(-15 + N(0, 2^2)); wall time of ``Engine.batch`` (host buffers in
    and out, best of ``repeats``)."""
    c = dataclasses.replace(cfg, vpm=dataclasses.replace(cfg.vpm, particle_cap=cap))
    eng = Engine.from_config(c)
    fl = FluidState.empty(c.vpm)
    x0 = np.array([0.0, 0.0, 0.3, 0.0, 7.0, 0.0, 0.0])
    lim = eng.params.u_limit
    rows = []
    for B in batches:
        u = np.clip(-15.0 + 2.0 * np.random.default_rng(seed + B).normal(0.0, 1.0, (B, horizon)), -lim, lim)
        req = RolloutRequest(x0=x0, fluid=fl, controls=u)
        res = eng.batch(req)  # warm-up (plan, scratch)
        times = []
        for _ in range(repeats):
            t0 = time.perf_counter()
            res = eng.batch(req)
            times.append(1e3 * (time.perf_counter() - t0))
        rows.append({"batch": int(B), "best_ms": min(times), "median_ms": float(np.median(times)),
                     "failed": int(np.count_nonzero(res.status))})
    return {"schema": SCHEMA, "config_hash": c.config_hash(), "horizon": horizon, "particle_cap": cap,
            "hardware_threads": os.cpu_count(), "rows": rows}


def _write_rows_csv(rows, path: str, cfg_hash: str) -> None:
    keys = list(rows[0].keys()) if rows else []
    with open(path, "w") as fh:
        fh.write(f"# config_hash={cfg_hash} schema={SCHEMA}\n")
        fh.write(",".join(keys) + "\n")
        for r in rows:
            fh.write(",".join(str(r[k]) for k in keys) + "\n")


def _load(path: str | None) -> ExperimentConfig:
    if path is None:
        cfg = ExperimentConfig()
        cfg.validate()
        return cfg
    return config_mod.load_config(path)


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_2509_16079_b200", description=__doc__.splitlines()[0])
    sub = ap.add_subparsers(dest="cmd", required=True)
    p = sub.add_parser("trial", help="closed-loop perching trials")
    p.add_argument("--config")
    p.add_argument("--mode", default="all", help="|".join(MODES) + "|all")
    p.add_argument("--trials", type=int)
    p.add_argument("--seed", type=int)
    p.add_argument("--out")
    p = sub.add_parser("sweep", help="initial-condition sweep, open loop vs TVLQR")
    p.add_argument("--config")
    p.add_argument("--state", type=int, default=5, help="1-based state index (5 = v_x)")
    p.add_argument("--lo", type=float, default=-0.3)
    p.add_argument("--hi", type=float, default=0.3)
    p.add_argument("--steps", type=int, default=7)
    p.add_argument("--seed", type=int)
    p.add_argument("--out")
    p = sub.add_parser("bench", help="batch-runtime table")
    p.add_argument("--config")
    p.add_argument("--batches", default="1,128,256,512,1024")
    p.add_argument("--horizon", type=int, default=80)
    p.add_argument("--cap", type=int, default=60)
    p.add_argument("--repeats", type=int, default=5)
    p.add_argument("--out")
    p = sub.add_parser("validate-config", help="schema-check a config file")
    p.add_argument("--config", required=True)
    a = ap.parse_args(argv)
    try:
        cfg = _load(a.config)
    except (ConfigError, ValueError, OSError) as e:
        print(f"config error: {e}", file=sys.stderr)
        return 2
    if a.cmd == "validate-config":
        print(json.dumps({"valid": True, "config_hash": cfg.config_hash()}))
        return 0
    if a.cmd == "trial":
        modes = MODES if a.mode == "all" else (a.mode,)
        summary, recs = run_trials(cfg, modes, a.trials or cfg.trials, a.seed, a.out)
        print(json.dumps(summary, sort_keys=True))
        return 0 if all(r.failure is None for rs in recs.values() for r in rs) else 1
    if a.cmd == "sweep":
        res = run_sweep(cfg, a.state, a.lo, a.hi, a.steps, a.seed)
        if a.out:
            os.makedirs(a.out, exist_ok=True)
            _write_rows_csv(res["rows"], os.path.join(a.out, "sweep.csv"), res["config_hash"])
        print(json.dumps(res))
        return 0
    res = run_bench(cfg, tuple(int(b) for b in a.batches.split(",")), a.horizon, a.cap, a.repeats)
    if a.out:
        os.makedirs(a.out, exist_ok=True)
        _write_rows_csv(res["rows"], os.path.join(a.out, "bench.csv"), res["config_hash"])
    print(json.dumps(res))
    return 0


if __name__ == "__main__":
    sys.exit(main())
