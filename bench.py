#!/usr/bin/env python
"""bench.py -- MPPI replanning iteration of the VPM perching planner on B200.

Workload (BASELINE.json config C4): one MPPI iteration = K=4096 sampled control
sequences + the incumbent (B=4097 rollouts), H=50 coupled glider + vortex-wake
steps each, particle cap N=512 on a prefilled synthetic wake (510 particles,
reference-generated fixture tests/golden/scenario_C4.npz) plus the planarised
ring-vortex pair; x0=[0,0,0.3,0,7,0,0], warm start -6 rad/s, sigma=2, lambda=0.05,
noise = numpy default_rng(seed).normal(0, 1, (K, H)) per iteration.

  value        rollouts/s of the whole job (B x steps / device time, max over ranks)
  ms_per_step  MPPI iteration latency (device, CUDA events on the launch stream)
  e2e          same metric through the C ABI with host buffers (vpm_plan_set_fluid +
               vpm_mppi_optimize_host: H2D of snapshot/noise/u*, D2H of u*)
  roofline     rollout kernel vs the FP32 CUDA-core peak (12 flop per directed
               regularised Biot-Savart interaction, counted exactly by the kernel)

``--impl reference`` times the reference's own compiled CPU core
(oracle/_ref, Cython + OpenMP FP64, all host threads) on a bounded sample of the
same workload, driven by the numpy restatement of mppi.py.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

K_SAMPLES, HORIZON, CAP = 4096, 50, 512
SIGMA, LAMBDA = 2.0, 0.05
Q = [10.0, 10.0, 1.0, 0.0, 0.2, 0.2, 0.2]
XPERCH = [3.5, 0.0, np.pi / 4.0, 0.0, 0.5, -0.5, 0.0]
FP32_SPEC_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12  # 74.4, SMs x lanes x FMA x max clock
METRIC = "MPPI iteration rollouts/s (K=4096, H=50, N<=512 + ring)"
CONFIG = {"workload": "C4: MPPI perching + ring vortex, K=4096 (+incumbent), H=50, N<=512",
          "K": K_SAMPLES, "H": HORIZON, "particle_cap": CAP, "n_bound": 10,
          "scenario": "tests/golden/scenario_C4.npz (reference-generated prefilled wake + ring)",
          "l2": "flushed (256 MiB write) before every timed iteration"}


def load_scenario():
    with np.load(os.path.join(ROOT, "tests", "golden", "scenario_C4.npz")) as z:
        sc = {k: z[k] for k in z.files}
    flat = (sc["wake_pos"], sc["wake_gamma"], sc["wake_age"], int(sc["n_wake"]), int(sc["ring_a"]),
            int(sc["ring_b"]), sc["prev_pos"], sc["prev_gamma"], int(sc["n_prev"]),
            float(sc["prev_lev"]), sc["ema"])
    return sc, flat


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self._proc = None

    def __enter__(self):
        # one streaming nvidia-smi (-lms 50) for the whole timed region
        try:
            self._proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            time.sleep(0.3)  # let it attach before the timed region starts
        except Exception:
            self._proc = None
        return self

    def __exit__(self, *a):
        if self._proc is None:
            return
        time.sleep(0.1)
        self._proc.terminate()
        try:
            out, _ = self._proc.communicate(timeout=5)
        except Exception:
            self._proc.kill()
            out = ""
        for line in (out or "").splitlines():
            parts = [c.strip() for c in line.split(",")]
            if len(parts) >= 7:
                self.rows.append(parts)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        reasons = sorted({n for r in self.rows for n, v in zip(names, r[3:7]) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def read_traffic():
    """DRAM bytes per rollout-kernel launch from the committed ncu --set full capture."""
    p = os.path.join(ROOT, "profiles", "rollout_kernel_ncu.json")
    if os.path.exists(p):
        with open(p) as fh:
            return json.load(fh).get("dram_bytes_per_launch")
    return None


# ------------------------------------------------------------------------------ CPU arm
def reference_core():
    from oracle import refcore
    mod = refcore.load()
    if mod is not None:
        return mod, "reference"
    from oracle import core
    core.build()
    return core, "port"


def time_cpu_sample(core, sc, flat, noise, rows):
    """Run ``rows`` candidate rows of the C4 iteration on the host; returns seconds."""
    from oracle import planner
    cand = planner.candidates(np.full(HORIZON, -6.0), noise[: rows - 1], SIGMA, 15.0)
    threads = os.cpu_count() or 1
    t0 = time.perf_counter()
    status, finals, _ = core.batch_rollout(sc["x0"], np.ascontiguousarray(cand), *flat, sc["iparams"],
                                           sc["fparams"], False, threads)
    J = planner.terminal_costs(finals, status, Q, XPERCH)
    planner.weighted_mean(cand, J, LAMBDA)
    return time.perf_counter() - t0


def cpu_baseline(sc, flat):
    """The reference's CPU planner on one full C4 iteration (all 4097 candidate rows,
    same snapshot and noise shape as the GPU arm), all host threads."""
    core, kind = reference_core()
    noise = np.random.default_rng(1234).normal(0.0, 1.0, (K_SAMPLES, HORIZON))
    threads = os.cpu_count() or 1
    time_cpu_sample(core, sc, flat, noise, 2 * threads)  # warm the OpenMP pool
    dt = time_cpu_sample(core, sc, flat, noise, K_SAMPLES + 1)
    return {"value": (K_SAMPLES + 1) / dt, "unit": "rollouts/s", "cores": threads, "kind": kind,
            "sample": f"one full C4 MPPI iteration: all {K_SAMPLES + 1} candidate rollouts (H=50, N=512 + "
                      f"ring) + terminal costs + softmax update, FP64, {threads} OpenMP threads, {dt:.2f} s"}


def run_reference(args):
    """--impl reference: the reference's own compiled CPU core (oracle/_ref), full C4
    iterations (4097 rollouts + costs + update) per timed step -- no extrapolation.
    Warm-up steps run a small slice (OpenMP pool and page cache only)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    sc, flat = load_scenario()
    core, kind = reference_core()
    noise = np.random.default_rng(1234).normal(0.0, 1.0, (K_SAMPLES, HORIZON))
    threads = os.cpu_count() or 1
    for _ in range(max(args.warmup, 1)):
        time_cpu_sample(core, sc, flat, noise, 2 * threads)
    times = [time_cpu_sample(core, sc, flat, noise, K_SAMPLES + 1) for _ in range(args.steps)]
    tot = sum(times)
    value = (K_SAMPLES + 1) * args.steps / tot
    line = {"metric": METRIC, "value": value, "unit": "rollouts/s", "impl": "reference",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * tot / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": CONFIG,
            "cpu_baseline": {"value": value, "unit": "rollouts/s", "cores": threads, "kind": kind,
                             "sample": f"full C4 iterations ({K_SAMPLES + 1} rollouts each), "
                                       f"{args.steps} timed, {min(times):.2f}-{max(times):.2f} s each"},
            "e2e": {"value": value, "unit": "rollouts/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def cpu_baselines_other_configs():
    """Same-run CPU baselines for the other BASELINE.json configs, on the reference's
    compiled core (oracle/_ref, all host threads) -- C2 and C3 as full iterations,
    C5 on a K-subset extrapolated linearly in K (labelled) -- and, past the compiled
    core's MAXW = 1028 (C5 N = 2048), the reference's numpy induced_velocity_at
    (vpm.py:105-128) on a K-subset, extrapolated."""
    from oracle import planner
    core, kind = reference_core()
    threads = os.cpu_count() or 1
    out = {"cores": threads, "kind": kind}
    for tag, name, K in (("C2", "scenario_C2.npz", 256), ("C3", "scenario_C3.npz", 1024)):
        with np.load(os.path.join(ROOT, "tests", "golden", name)) as z:
            s = {k: z[k] for k in z.files}
        fl = (s["wake_pos"], s["wake_gamma"], s["wake_age"], int(s["n_wake"]), int(s["ring_a"]), int(s["ring_b"]),
              s["prev_pos"], s["prev_gamma"], int(s["n_prev"]), float(s["prev_lev"]), s["ema"])
        cand = np.ascontiguousarray(planner.candidates(np.full(HORIZON, -6.0),
                                                       np.random.default_rng(7).normal(0, 1, (K, HORIZON)),
                                                       SIGMA, 15.0))
        core.batch_rollout(s["x0"], cand[: 2 * threads], *fl, s["iparams"], s["fparams"], False, threads)
        t0 = time.perf_counter()
        st, fin, _ = core.batch_rollout(s["x0"], cand, *fl, s["iparams"], s["fparams"], False, threads)
        planner.weighted_mean(cand, planner.terminal_costs(fin, st, Q, XPERCH), LAMBDA)
        dt = time.perf_counter() - t0
        out[tag] = {"iteration_ms": 1e3 * dt, "rollouts_per_s": (K + 1) / dt,
                    "sample": f"full iteration, {K + 1} rollouts"}
    from paper_2509_16079_b200 import config
    c5 = {}
    K5, H5 = 16384, 5
    for N in (128, 256, 512, 1024, 2048):
        rng = np.random.default_rng(11)
        v = config.VpmConfig(particle_cap=N)
        ip, fp = config.pack_params(v, config.GliderParams())
        wp = rng.normal(0.0, 0.5, (N, 2))
        wp[:, 0] -= 3.0
        g = rng.normal(0.0, 0.05, N)
        inter = N * (N - 1) + 10 * N * 3  # wake-wake + bound row + collocation + loads (no shedding)
        if N <= 1024:
            fl = (wp, g, np.zeros(N, np.int64), N, -1, -1, np.zeros((10, 2)), np.zeros(10), 0, 0.0, np.zeros(10))
            x0 = np.array([0.0, 0.0, 0.0, 0.0, 7.0, 0.0, 0.0])
            sub = max(threads, min(K5, int(2e9 / (N * N * H5))))  # ~1-2 s of work
            sub = (sub // threads) * threads
            ctrl = np.zeros((sub, H5))
            core.batch_rollout(x0, ctrl[:threads], *fl, ip, fp, False, threads)
            t0 = time.perf_counter()
            core.batch_rollout(x0, ctrl, *fl, ip, fp, False, threads)
            dt = time.perf_counter() - t0
            c5[str(N)] = {"ms_extrapolated_K16384": 1e3 * dt * K5 / sub, "sample_rollouts": sub,
                          "gflops": 12.0 * inter * H5 * sub / dt / 1e9,
                          "sample": f"{sub} of {K5} rollouts x {H5} steps on the compiled core, "
                                    "extrapolated linearly in K"}
        else:
            from oracle import refpkg
            if not refpkg.available():
                c5[str(N)] = {"unavailable": "reference package not staged (oracle/build_ref.sh)"}
                continue
            refpkg.load()
            import importlib
            vpm_ref = importlib.import_module("perchsim.vpm")
            reps = 3
            t0 = time.perf_counter()
            for _ in range(reps):  # one rollout-step's wake-wake sum, the O(N^2) part
                vpm_ref.induced_velocity_at(wp, wp, g, vpm_ref.KERNEL_REGULARIZED, 0.02)
            dt = (time.perf_counter() - t0) / reps
            c5[str(N)] = {"ms_extrapolated_K16384": 1e3 * dt * K5 * H5, "sample_rollout_steps": reps,
                          "gflops": 12.0 * N * N / dt / 1e9,
                          "sample": "numpy induced_velocity_at (vpm.py:105-128) of one 2048-particle wake "
                                    "on itself, 1 thread, extrapolated to K=16384 x H=5 (compiled core "
                                    "limited to N <= 1024 by MAXW)"}
    out["C5"] = {"K": K5, "H": H5, "by_N": c5}
    return out


# ------------------------------------------------------------------------------ GPU arm
def _time_ms(torch, fn, reps=3):
    fn()
    torch.cuda.synchronize()
    best = float("inf")
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    return best


def _b2b_ms(torch, fn, reps=10):
    """Device time per call of ``reps`` back-to-back calls (CUDA events around the
    batch; the host enqueues ahead of the GPU, so no launch gap enters), best of 3."""
    fn()
    torch.cuda.synchronize()
    best = float("inf")
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            fn()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) / reps)
    return best


def extras(torch, dev, sc, flat, plan, mp):
    """Side measurements (not the headline): the C2 latency config, policy
    synthesis on the C4 snapshot, and the C5 Biot-Savart stress sweep."""
    from paper_2509_16079_b200 import config, policy, rollout, vpm
    from paper_2509_16079_b200.device import DevicePlan
    f64 = lambda a: torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64), device=dev)
    out = {}
    # C2: K=256 (+1), H=50, cap 60, empty fluid -- latency-bound configuration
    with np.load(os.path.join(ROOT, "tests", "golden", "scenario_C2.npz")) as z:
        s2 = {k: z[k] for k in z.files}
    p2 = DevicePlan(s2["iparams"], s2["fparams"], device=dev.index)
    p2.set_fluid((s2["wake_pos"], s2["wake_gamma"], s2["wake_age"], 0, -1, -1, s2["prev_pos"],
                  s2["prev_gamma"], 0, 0.0, s2["ema"]))
    n2 = f64(np.random.default_rng(5).normal(0, 1, (256, HORIZON)))
    sc2 = {"cost": torch.empty(257, dtype=torch.float64, device=dev),
           "partial": torch.empty(HORIZON + 2, dtype=torch.float64, device=dev),
           "flag": torch.zeros(1, dtype=torch.int32, device=dev)}
    u2 = f64(np.full(HORIZON, -6.0))
    x2, q_d, xp_d = f64(s2["x0"]), f64(Q), f64(XPERCH)
    # device time of one iteration (rollouts + fused softmax update), iterations back to back
    out["c2_iteration_ms"] = _b2b_ms(torch, lambda: p2.mppi_iteration(
        x2, u2, n2, SIGMA, 257, LAMBDA, q_d, xp_d, sc2))
    # C3: K=1024 (+1), H=50, N<=256 + ring (reference-generated prefilled wake)
    with np.load(os.path.join(ROOT, "tests", "golden", "scenario_C3.npz")) as z:
        s3 = {k: z[k] for k in z.files}
    p3 = DevicePlan(s3["iparams"], s3["fparams"], device=dev.index)
    p3.set_fluid((s3["wake_pos"], s3["wake_gamma"], s3["wake_age"], int(s3["n_wake"]), int(s3["ring_a"]),
                  int(s3["ring_b"]), s3["prev_pos"], s3["prev_gamma"], int(s3["n_prev"]), float(s3["prev_lev"]),
                  s3["ema"]))
    n3 = f64(np.random.default_rng(6).normal(0, 1, (1024, HORIZON)))
    sc3 = {"cost": torch.empty(1025, dtype=torch.float64, device=dev),
           "partial": torch.empty(HORIZON + 2, dtype=torch.float64, device=dev),
           "flag": torch.zeros(1, dtype=torch.int32, device=dev)}
    u3, x3 = f64(np.full(HORIZON, -6.0)), f64(s3["x0"])
    ms3 = _b2b_ms(torch, lambda: p3.mppi_iteration(x3, u3, n3, SIGMA, 1025, LAMBDA, q_d, xp_d, sc3))
    out["c3_iteration"] = {"ms": ms3, "rollouts_per_s": 1025 / (ms3 * 1e-3),
                           "config": "C3: K=1024 (+incumbent), H=50, N<=256 + ring, 1 GPU"}
    # one rank's share of the C4 iteration at 8 GPUs (rows [0, 513) of 4097): its
    # rollouts, its softmax partial and the rank-ordered combine (a W = 1 stand-in for
    # the W = 8 combine; the all-gather of 8 x (H+2) doubles is not on one GPU)
    from paper_2509_16079_b200.device import mppi_combine
    from paper_2509_16079_b200.sharding import row_range
    b8, e8 = row_range(mp.B, 8, 0)
    o8 = {"status": torch.empty(e8 - b8, dtype=torch.int64, device=dev),
          "finals": torch.empty(e8 - b8, 7, dtype=torch.float64, device=dev),
          "cost": torch.empty(e8 - b8, dtype=torch.float64, device=dev)}
    part8, flag8 = torch.empty(mp.T + 2, dtype=torch.float64, device=dev), torch.zeros(1, dtype=torch.int32,
                                                                                       device=dev)
    us8 = mp.ustar.clone()
    u8 = us8.clone()

    def rank_share():
        plan.batch(mp.x0, mp.T, ustar=us8, noise=mp.noise, sigma=mp.sigma, row_begin=b8, rows=e8 - b8, q=mp.q,
                   x_perch=mp.xp, out=o8)
        plan.mppi_partial(o8["cost"], us8, mp.noise, mp.sigma, mp.temperature, row_begin=b8, partial=part8)
        mppi_combine(part8.view(1, -1), mp.temperature, u8, flag8)

    ms8 = _b2b_ms(torch, rank_share)
    out["c4_rank_share_8gpu"] = {"rows": e8 - b8, "ms": ms8, "expected_8gpu_iteration_ms": ms8 + 0.05,
                                 "note": "rank 0's rows of the C4 batch at world 8 + its partial + combine, "
                                         "device-timed back to back on one GPU; + <=0.05 ms all-gather "
                                         "(DESIGN.md 5)"}
    # policy synthesis (64 perturbed rollouts on the N=512 + ring snapshot, regression,
    # Riccati) through the C ABI with host buffers, around the current u*
    cfg = config.ExperimentConfig()
    cfg.vpm.particle_cap = CAP
    eng = rollout.Engine(cfg.vpm, cfg.glider)
    eng._device_plan = plan
    fl = vpm.FluidState.empty(cfg.vpm)
    n = int(sc["n_wake"])
    fl.wake_pos[:n], fl.wake_gamma[:n], fl.wake_age[:n] = sc["wake_pos"][:n], sc["wake_gamma"][:n], sc["wake_age"][:n]
    fl.n_wake, fl.ring_a, fl.ring_b = n, int(sc["ring_a"]), int(sc["ring_b"])
    fl.prev_pos[:], fl.prev_gamma[:], fl.n_prev = sc["prev_pos"], sc["prev_gamma"], int(sc["n_prev"])
    fl.prev_lev_gamma, fl.unsteady_ema[:] = float(sc["prev_lev"]), sc["ema"]
    u_nom = mp.ustar.cpu().numpy()
    rc, traj, _ = eng.rollout(sc["x0"], u_nom, fl, record=True)
    if rc == 0:
        nom = policy.NominalTrajectory(states=traj, inputs=u_nom, dt=cfg.vpm.dt)
        policy.build_policy(nom, fl, cfg.synthesis, eng, np.random.default_rng(0))
        t0 = time.perf_counter()
        for i in range(3):
            policy.build_policy(nom, fl, cfg.synthesis, eng, np.random.default_rng(i))
        out["policy_build_ms_e2e"] = 1e3 * (time.perf_counter() - t0) / 3
    # mppi.optimize through the public API on the C4 snapshot (K=4096, H=50, 3
    # iterations, host buffers in/out): numpy noise drawn on the host (reference
    # parity; iteration i+1's draw overlaps iteration i) vs device-drawn Philox noise
    import dataclasses
    from paper_2509_16079_b200 import mppi as mppi_mod
    mcfg = dataclasses.replace(cfg.mppi, batch=K_SAMPLES, input_stdev=SIGMA, temperature=LAMBDA)
    warm = np.full(HORIZON, -6.0)
    for name, mk in (("numpy_rng", lambda i: np.random.default_rng(i)),
                     ("device_noise", lambda i: mppi_mod.DeviceNoise(i))):
        mppi_mod.optimize(sc["x0"], fl, warm, mcfg, eng, mk(0), iterations=3)
        t0 = time.perf_counter()
        for i in range(3):
            mppi_mod.optimize(sc["x0"], fl, warm, mcfg, eng, mk(1 + i), iterations=3)
        out[f"optimize_c4_3iter_ms_{name}"] = 1e3 * (time.perf_counter() - t0) / 3
    plan.set_fluid(flat)
    # one full replanning cycle at the paper's operating point (nmpc.replan: 10-step
    # projection, 3 MPPI iterations K=256 over the 67-step tail, nominal, policy; cap 60)
    from paper_2509_16079_b200 import replan as rp
    from paper_2509_16079_b200.policy import NominalTrajectory, Policy
    with np.load(os.path.join(ROOT, "tests", "golden", "nmpc_replan.npz")) as z:
        gr = {k: z[k] for k in z.files}
    cfg_r = config.ExperimentConfig()
    eng_r = rollout.Engine.from_config(cfg_r)
    pol = Policy(gains=gr["boot_gains"], nominal=NominalTrajectory(gr["boot_states"], gr["boot_inputs"], 0.01))
    req = rp.ReplanRequest(x=np.asarray(cfg_r.scenario.x0, float), fluid=vpm.FluidState.empty(cfg_r.vpm),
                           policy=pol, t=0.0, t_proj=10)
    rp.replan(req, cfg_r, eng_r, np.random.default_rng(1))
    t0 = time.perf_counter()
    for i in range(3):
        rp.replan(req, cfg_r, eng_r, np.random.default_rng(1 + i))
    out["replan_cycle_ms_e2e"] = 1e3 * (time.perf_counter() - t0) / 3
    rp.replan(req, cfg_r, eng_r, mppi_mod.DeviceNoise(0))
    t0 = time.perf_counter()
    for i in range(3):
        rp.replan(req, cfg_r, eng_r, mppi_mod.DeviceNoise(1 + i))
    out["replan_cycle_ms_e2e_device_noise"] = 1e3 * (time.perf_counter() - t0) / 3
    # C5: Biot-Savart stress sweep, K=16384 rollouts, attached flow (no shedding, fixed N)
    sweep = {}
    rng = np.random.default_rng(11)
    K5, H5 = 16384, 5
    for N in (128, 256, 512, 1024, 2048):
        v = config.VpmConfig(particle_cap=N)
        ip, fp = config.pack_params(v, config.GliderParams())
        p5 = DevicePlan(ip, fp, device=dev.index)
        wp = rng.normal(0.0, 0.5, (N, 2))
        wp[:, 0] -= 3.0  # wake behind the plate, plate at the origin
        p5.set_fluid((wp, rng.normal(0.0, 0.05, N), np.zeros(N, np.int64), N, -1, -1,
                      np.zeros((10, 2)), np.zeros(10), 0, 0.0, np.zeros(10)))
        x5 = f64([0.0, 0.0, 0.0, 0.0, 7.0, 0.0, 0.0])
        ctrl = torch.zeros(K5, H5, dtype=torch.float64, device=dev)
        o5 = {"status": torch.empty(K5, dtype=torch.int64, device=dev),
              "finals": torch.empty(K5, 7, dtype=torch.float64, device=dev),
              "interactions": torch.zeros(K5, dtype=torch.int64, device=dev)}
        ms = _time_ms(torch, lambda: p5.batch(x5, H5, controls=ctrl, rows=K5, out=o5))
        inter = float(o5["interactions"].sum().item())
        shed = int((o5["status"] != 0).sum().item())
        sweep[str(N)] = {"ms": ms, "interactions": inter,
                         "gflops": 12.0 * inter / (ms * 1e-3) / 1e9,
                         "frac_of_fp32_peak": 12.0 * inter / (ms * 1e-3) / 1e12 / FP32_SPEC_TFLOPS,
                         "failed_rollouts": shed}
    out["single_instance_stepping"] = step_latency(torch)
    out["c5_biot_savart_sweep"] = {"K": K5, "H": H5, "by_N": sweep,
                                   "note": "random wake pos~N(0,0.5^2), Gamma~N(0,0.05^2), "
                                           "attached flow; 12 flop per directed interaction"}
    return out


def step_latency(torch):
    """Single-instance stepping (rollout.py:81-98, called every tick at nmpc.py:314-315):
    per-call latency of Engine.step / fluid_step through the reference stepping
    contract with host buffers (the C ABI's vpm_step), of the device-resident step
    (plant.DeviceWake: x up, a small record back, the fluid stays on the device),
    of one resident control-loop tick (plant step + sensor + observed-wake step, one
    sync), and of the reference's compiled core step on this host (oracle/_ref,
    FP64, 1 thread per call) -- at cap 60 (the closed-loop default, ~60-particle
    wake) and cap 512 (the C4 N=512 + ring snapshot)."""
    from paper_2509_16079_b200 import config, rollout, vpm
    from paper_2509_16079_b200.plant import DeviceWake
    core, kind = reference_core()
    x0 = np.array([0.0, 0.0, 0.3, 0.0, 7.0, 0.0, 0.0])
    res = {"reference_kind": kind}
    for cap in (60, 512):
        cfg = config.ExperimentConfig()
        cfg.vpm.particle_cap = cap
        eng = rollout.Engine(cfg.vpm, cfg.glider)
        if cap == 512:
            sc, _ = load_scenario()
            fl = vpm.FluidState.empty(cfg.vpm)
            n = int(sc["n_wake"])
            fl.wake_pos[:n], fl.wake_gamma[:n], fl.wake_age[:n] = sc["wake_pos"][:n], sc["wake_gamma"][:n], sc["wake_age"][:n]
            fl.n_wake, fl.ring_a, fl.ring_b = n, int(sc["ring_a"]), int(sc["ring_b"])
            fl.prev_pos[:], fl.prev_gamma[:], fl.n_prev = sc["prev_pos"], sc["prev_gamma"], int(sc["n_prev"])
            fl.prev_lev_gamma, fl.unsteady_ema[:] = float(sc["prev_lev"]), sc["ema"]
        else:
            fl, xx = vpm.FluidState.empty(cfg.vpm), x0.copy()
            for _ in range(40):  # prefill to the cap through the plant itself
                _, xx, fl, _ = eng.step(xx, -15.0, fl)
        reps = 200

        def timed(fn):
            for _ in range(10):
                fn()
            t0 = time.perf_counter()
            for _ in range(reps):
                fn()
            return 1e6 * (time.perf_counter() - t0) / reps

        r = {"n_wake": int(fl.n_wake)}
        r["engine_step_us"] = timed(lambda: eng.step(x0, -6.0, fl))
        r["engine_fluid_step_us"] = timed(lambda: eng.fluid_step(x0, fl))
        dw = DeviceWake(eng, fl)
        ob = DeviceWake(eng, fl)

        def resident_step():
            dw.step_async(x0, -6.0, True)
            dw.sync()
            return dw.record()

        def resident_tick():
            dw.step_async(x0, -6.0, True, sensor=(1.0, 0.3), r_core=cfg.vpm.r_core)
            ob.step_async(x0, 0.0, False)
            dw.sync()
            ob.sync()
            return dw.record(), ob.record()

        r["resident_step_us"] = timed(resident_step)
        r["resident_loop_tick_us"] = timed(resident_tick)
        ip, fp = eng.iparams, eng.fparams
        flat = fl.flat()
        r["reference_core_step_us"] = timed(lambda: core.step(x0, -6.0, *flat, ip, fp, True))
        res[f"cap{cap}"] = r
    return res


def c5_sharded(torch, dev, rank, world):
    """C5 (Biot-Savart stress, K=16384 rollouts x H=5, attached flow) with the
    rollouts sharded over the ranks; device time max over ranks, interactions
    summed; fraction of world x FP32 peak."""
    import torch.distributed as dist
    from paper_2509_16079_b200 import config
    from paper_2509_16079_b200.device import DevicePlan
    from paper_2509_16079_b200.sharding import row_range
    K5, H5 = 16384, 5
    b, e = row_range(K5, world, rank)
    res = {}
    for N in (512, 2048):
        rng = np.random.default_rng(1000 + N)  # same wake on every rank
        v = config.VpmConfig(particle_cap=N)
        ip, fp = config.pack_params(v, config.GliderParams())
        p5 = DevicePlan(ip, fp, device=dev.index)
        wp = rng.normal(0.0, 0.5, (N, 2))
        wp[:, 0] -= 3.0
        p5.set_fluid((wp, rng.normal(0.0, 0.05, N), np.zeros(N, np.int64), N, -1, -1,
                      np.zeros((10, 2)), np.zeros(10), 0, 0.0, np.zeros(10)))
        x5 = torch.tensor([0.0, 0.0, 0.0, 0.0, 7.0, 0.0, 0.0], dtype=torch.float64, device=dev)
        ctrl = torch.zeros(e - b, H5, dtype=torch.float64, device=dev)
        o5 = {"status": torch.empty(e - b, dtype=torch.int64, device=dev),
              "finals": torch.empty(e - b, 7, dtype=torch.float64, device=dev),
              "interactions": torch.zeros(e - b, dtype=torch.int64, device=dev)}
        ms = _time_ms(torch, lambda: p5.batch(x5, H5, controls=ctrl, rows=e - b, out=o5))
        st = torch.tensor([ms, float(o5["interactions"].sum().item())], dtype=torch.float64, device=dev)
        if world > 1:
            mx, sm = st.clone(), st.clone()
            dist.all_reduce(mx, op=dist.ReduceOp.MAX)
            dist.all_reduce(sm, op=dist.ReduceOp.SUM)
            ms, inter = float(mx[0]), float(sm[1])
        else:
            inter = float(st[1])
        tf = 12.0 * inter / (ms * 1e-3) / 1e12
        res[str(N)] = {"ms": ms, "tflops": tf, "frac_of_fp32_peak": tf / (world * FP32_SPEC_TFLOPS),
                       "rows_per_rank": e - b}
    return {"K": K5, "H": H5, "n_gpus": world, "by_N": res}


def run_ours(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # functional-test hooks (never set by the driver): every rank on device 0 and
    # gloo instead of NCCL, to exercise the multi-rank code path on a 1-GPU box
    if os.environ.get("VPM_BENCH_ONE_DEVICE"):
        local = 0
    backend = os.environ.get("VPM_BENCH_BACKEND", "nccl")
    torch.cuda.set_device(local)
    if world > 1:
        if backend == "nccl":
            # NCCL's communicator setup lines (nranks, NVLS / P2P transports) go to
            # stderr, so a run's log shows that N ranks formed one communicator
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
        if rank == 0:
            ver = torch.cuda.nccl.version() if backend == "nccl" else None
            print(f"bench: {world} ranks, backend {backend}, NCCL {ver}", file=sys.stderr, flush=True)
    from paper_2509_16079_b200 import _lib
    from paper_2509_16079_b200.device import DevicePlan, fp32_peak_gflops, launch_shape
    from paper_2509_16079_b200.sharding import ShardedMppi

    sc, flat = load_scenario()
    dev = torch.device("cuda", local)
    f64 = lambda a: torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64), device=dev)
    B = K_SAMPLES + 1
    plan = DevicePlan(sc["iparams"], sc["fparams"], device=local)
    plan.set_fluid(flat)
    nsteps = args.warmup + args.steps
    noise_all = [f64(np.random.default_rng(100 + i).normal(0.0, 1.0, (K_SAMPLES, HORIZON)))
                 for i in range(nsteps)]
    warm = f64(np.full(HORIZON, -6.0))
    mp = ShardedMppi(plan, f64(sc["x0"]), warm, noise_all[0], B=B, sigma=SIGMA, temperature=LAMBDA,
                     q=f64(Q), x_perch=f64(XPERCH), rank=rank, world=world)
    mp.out["interactions"] = torch.zeros(mp.end - mp.begin, dtype=torch.int64, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream()

    for i in range(args.warmup):
        mp.set_noise(noise_all[i])
        mp.iteration()
    torch.cuda.synchronize()
    mp.check()

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    inter_total = 0
    plan.timing(reset=1)  # start CUDA-event timing of every rollout launch
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for s in range(args.steps):
            flush.zero_()
            mp.set_noise(noise_all[args.warmup + s])
            ev[s][0].record(stream)
            mp.iteration()
            ev[s][1].record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    kern_ms, launches = plan.timing(reset=-1)
    mp.check()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    tot_ms = float(sum(step_ms))
    inter_total = int(mp.out["interactions"].sum().item())  # last iteration's count
    stats = torch.tensor([tot_ms, kern_ms, float(inter_total)], dtype=torch.float64, device=dev)
    if world > 1:
        mx = stats.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        sm = stats.clone()
        dist.all_reduce(sm, op=dist.ReduceOp.SUM)
        tot_ms, kern_ms_max, inter_all = float(mx[0]), float(mx[1]), float(sm[2])
    else:
        kern_ms_max, inter_all = kern_ms, float(inter_total)
    ms_per_step = tot_ms / args.steps
    value = B * args.steps / (tot_ms * 1e-3)

    # ---- end to end through the C ABI with host buffers (rank-local, 1 GPU)
    e2e = None
    if world == 1:
        import ctypes as C
        from paper_2509_16079_b200._lib import _D, VpmFluid, check, fluid_struct, ptr
        pin = torch.empty((args.steps, K_SAMPLES, HORIZON), dtype=torch.float64).pin_memory()
        pin_np = pin.numpy()
        for s in range(args.steps):
            pin_np[s] = noise_all[args.warmup + s].cpu().numpy()
        u_host = torch.empty(HORIZON, dtype=torch.float64).pin_memory().numpy()
        x0h = np.ascontiguousarray(sc["x0"])
        qh, xph = np.asarray(Q, float), np.asarray(XPERCH, float)
        L = _lib.lib()
        fstruct, keep = fluid_struct(*flat)

        split = [0.0, 0.0]

        def one(s):
            u_host[:] = -6.0
            t_a = time.perf_counter()
            check(L.vpm_plan_set_fluid(plan.handle, C.byref(fstruct)), "set_fluid")
            t_b = time.perf_counter()
            check(L.vpm_mppi_optimize_host(plan.handle, ptr(x0h, _D), ptr(u_host, _D),
                                           ptr(pin_np[s], _D), 1, K_SAMPLES, HORIZON, SIGMA, LAMBDA,
                                           ptr(qh, _D), ptr(xph, _D)), "optimize_host")
            split[0] += t_b - t_a
            split[1] += time.perf_counter() - t_b

        one(0)
        split[:] = [0.0, 0.0]
        t0 = time.perf_counter()
        for s in range(args.steps):
            one(s)
        e2e_s = time.perf_counter() - t0
        h2d = K_SAMPLES * HORIZON * 8 + HORIZON * 8 + 3 * 7 * 8 + int(sc["n_wake"]) * 32 + 10 * 32
        e2e = {"value": B * args.steps / e2e_s, "unit": "rollouts/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": HORIZON * 8 + 4, "ms_per_step": 1e3 * e2e_s / args.steps,
               "set_fluid_ms": 1e3 * split[0] / args.steps,
               "optimize_ms": 1e3 * split[1] / args.steps}

    elif world > 1:
        # the sharded planner's public API with host buffers: every step copies this
        # rank's noise rows from pinned memory and reads u* back; wall time, max over ranks
        lo, hi = max(mp.begin - 1, 0), mp.end - 1  # noise row of global row g is g - 1
        pin = torch.empty((args.steps, hi - lo, HORIZON), dtype=torch.float64).pin_memory()
        for s in range(args.steps):
            pin[s].copy_(noise_all[args.warmup + s][lo:hi])
        dnoise = torch.zeros((K_SAMPLES, HORIZON), dtype=torch.float64, device=dev)
        u_back = torch.empty(HORIZON, dtype=torch.float64).pin_memory()

        def one_sh(s):
            dnoise[lo:hi].copy_(pin[s], non_blocking=True)
            mp.set_noise(dnoise)
            mp.iteration()
            u_back.copy_(mp.ustar)  # D2H of the step's result (synchronising)

        one_sh(0)
        dist.barrier()
        t0 = time.perf_counter()
        for s in range(args.steps):
            one_sh(s)
        dist.barrier()
        wall = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
        dist.all_reduce(wall, op=dist.ReduceOp.MAX)
        e2e_s = float(wall[0])
        e2e = {"value": B * args.steps / e2e_s, "unit": "rollouts/s",
               "h2d_bytes_per_step": K_SAMPLES * HORIZON * 8, "d2h_bytes_per_step": world * HORIZON * 8,
               "ms_per_step": 1e3 * e2e_s / args.steps,
               "path": "ShardedMppi per rank: pinned H2D of the rank's noise rows, iteration "
                       "(rollouts + partial + all_gather + combine), D2H of u*; max over ranks"}

    c5 = None if args.no_c5 else c5_sharded(torch, dev, rank, world)
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    nt, r, smem = launch_shape(CAP, 10, mp.end - mp.begin)
    peak_meas = fp32_peak_gflops() / 1e3
    peak = max(peak_meas, FP32_SPEC_TFLOPS)
    mix_ceiling = max(fp32_peak_gflops(4096, 3) for _ in range(2)) / 1e3  # FP32+MUFU mix probe
    flops_per_launch = 12.0 * inter_all / max(world, 1)
    achieved = flops_per_launch / (kern_ms_max * 1e-3) / 1e12 if kern_ms_max > 0 else None
    line = {
        "metric": METRIC, "value": value, "unit": "rollouts/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": CONFIG,
        "parallelism": f"rollout rows sharded over {world} GPU(s), 1 all_gather of W x (H+2) f64 per "
                       "iteration" if world > 1 else "1 GPU: rollout rows in one launch, no collective",
        "latency_ms": ms_per_step,
        "biot_savart_gflops": 12.0 * inter_all / (kern_ms_max * 1e-3) / 1e9 if kern_ms_max > 0 else None,
        "roofline": {"bound": "fp32", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": (achieved / peak) if achieved else None,
                     "traffic": read_traffic(),
                     "kernel": f"rollout_kernel<{nt},{r}> (one CTA per rollout, {smem} B smem, "
                               + ("symmetric-pair sweep: each wake pair once for both directions, "
                                  f"{nt // 32} tiles of 128 particles)"
                                  if CAP > 256 and os.environ.get("VPM_SYM", "1") != "0" else "direct sweep)"),
                     "flop_per_launch": flops_per_launch,
                     "kernel_ms": kern_ms_max,
                     "peak_source": f"max(FFMA probe {peak_meas:.1f}, spec 148x128x2x1.965GHz "
                                    f"{FP32_SPEC_TFLOPS:.1f}) TFLOP/s; MEASURED_PEAKS.json has no FP32 entry",
                     "formulation_ceiling": {
                         "value": mix_ceiling, "unit": "TFLOP/s", "frac_of_peak": mix_ceiling / peak,
                         "achieved_frac_of_ceiling": (achieved / mix_ceiling) if achieved else None,
                         "source": "probe of the direct kernel's instruction mix (8 FP32 lane-ops + "
                                   "1 MUFU.RSQ per interaction, independent chains, no loads)"}},
        "c5_sharded": c5,
        "gpu_launches": ShardedMppi.kernels_per_iteration * args.steps,
        "clocks": clk.summary(),
    }
    if e2e is not None:
        line["e2e"] = e2e
    if world == 1 and not args.no_extras:
        line["extras"] = extras(torch, dev, sc, flat, plan, mp)
    if world == 1 and not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline(sc, flat)
        if "extras" in line:
            line["extras"]["cpu_baselines"] = cpu_baselines_other_configs()
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-c5", action="store_true", help="skip the sharded C5 stress measurement")
    ap.add_argument("--no-extras", action="store_true",
                    help="skip the C2 / policy / C5 Biot-Savart sweep side measurements")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
