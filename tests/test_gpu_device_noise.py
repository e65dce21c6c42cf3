"""Performance-mode noise drawn on the device (vpm_noise_philox).

Not a reference-parity path (the reference draws numpy PCG64 normals, mppi.py:42);
what is checked: the draws are standard normal, deterministic, independent of how
the rows are sharded, and mppi.optimize(..., rng=DeviceNoise(seed)) is bitwise the
host-noise pipeline fed with the same numbers."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    assert torch.cuda.is_available()
    torch.cuda.set_device(0)
    return torch


def test_philox_noise_is_standard_normal_and_shard_independent(torch_cuda):
    torch = torch_cuda
    from paper_2509_16079_b200.device import noise_philox
    from paper_2509_16079_b200.sharding import ShardedMppi, row_range
    K, H = 4096, 50
    full = noise_philox(11, 0, torch.empty((K, H), dtype=torch.float64, device="cuda"))
    again = noise_philox(11, 0, torch.empty((K, H), dtype=torch.float64, device="cuda"))
    nxt = noise_philox(11, 1, torch.empty((K, H), dtype=torch.float64, device="cuda"))
    a = full.cpu().numpy()
    assert np.array_equal(a, again.cpu().numpy())
    assert abs(a.mean()) < 0.01 and abs(a.std() - 1.0) < 0.01
    assert abs(np.mean(a ** 4) - 3.0) < 0.05                   # Gaussian kurtosis
    assert abs(np.corrcoef(a[:, :-1].ravel(), a[:, 1:].ravel())[0, 1]) < 0.01
    assert not np.allclose(a, nxt.cpu().numpy())
    # odd horizon and a row slice drawn on its own equal the full draw
    odd = noise_philox(11, 0, torch.empty((K, 49), dtype=torch.float64, device="cuda")).cpu().numpy()
    assert np.isfinite(odd).all()
    part = noise_philox(11, 0, torch.empty((500, H), dtype=torch.float64, device="cuda"), row_begin=1000)
    assert np.array_equal(part.cpu().numpy(), a[1000:1500])
    # ShardedMppi.draw_noise: every rank fills its rows; the union is the W = 1 matrix
    union = torch.zeros((K, H), dtype=torch.float64, device="cuda")
    for r in range(3):
        sh = ShardedMppi.__new__(ShardedMppi)
        sh.begin, sh.end = row_range(K + 1, 3, r)
        sh.noise = union
        sh.draw_noise(11, 0)
    assert np.array_equal(union.cpu().numpy(), a)


class _Replay:
    """A numpy-Generator stand-in that returns pre-drawn blocks from normal()."""

    class _BG:
        state = None

    def __init__(self, blocks):
        self.blocks = list(blocks)
        self.bit_generator = self._BG()

    def normal(self, loc, scale, size):
        return self.blocks.pop(0)


def test_optimize_with_device_noise_equals_host_pipeline(torch_cuda):
    torch = torch_cuda
    from paper_2509_16079_b200 import config, mppi, rollout, vpm
    from paper_2509_16079_b200.device import noise_philox
    cfg = config.ExperimentConfig()
    eng = rollout.Engine.from_config(cfg)
    x0 = np.asarray(cfg.scenario.x0, float)
    fl = vpm.inject_ring(vpm.FluidState.empty(cfg.vpm),
                         vpm.RingDisturbance.from_speed([1.0, -0.1], 7.5, 0.28, 0.02, -1.0))
    warm = np.full(cfg.mppi.horizon, -6.0)
    dn = mppi.DeviceNoise(5)
    u_dev = mppi.optimize(x0, fl, warm, cfg.mppi, eng, dn, iterations=3)
    assert dn.iteration == 3
    K, H = cfg.mppi.batch, cfg.mppi.horizon
    blocks = [noise_philox(5, i, torch.empty((K, H), dtype=torch.float64, device="cuda")).cpu().numpy()
              for i in range(3)]
    u_host = mppi.optimize(x0, fl, warm, cfg.mppi, eng, _Replay(blocks), iterations=3)
    np.testing.assert_array_equal(u_dev, u_host)
    # the next call continues the stream (iterations 3, 4) and stays deterministic
    u2 = mppi.optimize(x0, fl, warm, cfg.mppi, eng, mppi.DeviceNoise(5, iteration=3), iterations=2)
    u3 = mppi.optimize(x0, fl, warm, cfg.mppi, eng, dn, iterations=2)
    np.testing.assert_array_equal(u2, u3)


def test_replan_with_device_noise(torch_cuda):
    """nmpc.replan in performance mode: a policy comes back, the same seed gives the
    same policy, and the noise counter advances by iterations + 2 (cloud dx0, du)."""
    import os

    from conftest import GOLDEN
    from paper_2509_16079_b200 import config, mppi, replan as rp, rollout, vpm
    from paper_2509_16079_b200.policy import NominalTrajectory, Policy
    with np.load(os.path.join(GOLDEN, "nmpc_replan.npz")) as z:
        gr = {k: z[k] for k in z.files}
    cfg = config.ExperimentConfig()
    eng = rollout.Engine.from_config(cfg)
    pol = Policy(gains=gr["boot_gains"], nominal=NominalTrajectory(gr["boot_states"], gr["boot_inputs"], 0.01))
    req = rp.ReplanRequest(x=np.asarray(cfg.scenario.x0, float), fluid=vpm.FluidState.empty(cfg.vpm),
                           policy=pol, t=0.0, t_proj=10)
    dn = mppi.DeviceNoise(9)
    a = rp.replan(req, cfg, eng, dn)
    assert dn.iteration == cfg.mppi.iterations + 2
    b = rp.replan(req, cfg, eng, mppi.DeviceNoise(9))
    assert a is not None and b is not None
    np.testing.assert_array_equal(a.gains, b.gains)
    np.testing.assert_array_equal(a.nominal.inputs, b.nominal.inputs)
    assert np.isfinite(a.gains).all() and np.abs(a.nominal.inputs).max() <= cfg.glider.u_limit
    c = rp.replan(req, cfg, eng, dn)  # next counter block: a different plan
    assert c is None or not np.array_equal(c.nominal.inputs, a.nominal.inputs)
    # wiring: the same draws fed through the host path (iterations MPPI blocks, then
    # the cloud's start perturbations dx0 (k, 7) -- scaled by state_stdev -- and
    # input perturbations du (k, H) -- scaled by input_stdev) give bitwise the same
    # policy as the device-drawn replan
    import torch
    from paper_2509_16079_b200.device import noise_philox
    K, iters, k = cfg.mppi.batch, cfg.mppi.iterations, cfg.synthesis.n_samples
    H = len(a.nominal.inputs)
    draw = lambda i, r, c: noise_philox(9, i, torch.empty((r, c), dtype=torch.float64, device="cuda")).cpu().numpy()
    blocks = [draw(i, K, H) for i in range(iters)] + [draw(iters, k, 7), draw(iters + 1, k, H)]
    rep = _Replay(blocks)
    h = rp.replan(req, cfg, eng, rep)
    assert h is not None and not rep.blocks  # every block consumed, in order
    np.testing.assert_array_equal(h.gains, a.gains)
    np.testing.assert_array_equal(h.nominal.inputs, a.nominal.inputs)
    np.testing.assert_array_equal(h.nominal.states, a.nominal.states)
    # a swapped wiring (dx0 <-> du roles) would not reproduce it
    bad = [draw(i, K, H) for i in range(iters)] + [draw(iters + 1, k, 7), draw(iters, k, H)]
    w = rp.replan(req, cfg, eng, _Replay(bad))
    assert w is None or not np.array_equal(w.gains, a.gains)


def test_replan_graph_replay_equals_eager(torch_cuda):
    """The device-noise replan captured as a CUDA graph and replayed gives bitwise
    the launch-by-launch cycle, for several seeds through one cached graph, and a
    second shape gets its own graph."""
    import os
    import time

    from conftest import GOLDEN
    from paper_2509_16079_b200 import config, mppi, replan as rp, rollout, vpm
    from paper_2509_16079_b200.policy import NominalTrajectory, Policy
    with np.load(os.path.join(GOLDEN, "nmpc_replan.npz")) as z:
        gr = {k: z[k] for k in z.files}
    cfg = config.ExperimentConfig()
    eng = rollout.Engine.from_config(cfg)
    pol = Policy(gains=gr["boot_gains"], nominal=NominalTrajectory(gr["boot_states"], gr["boot_inputs"], 0.01))
    x0 = np.asarray(cfg.scenario.x0, float)
    for t in (0.0, 0.1):
        req = rp.ReplanRequest(x=x0, fluid=vpm.FluidState.empty(cfg.vpm), policy=pol, t=t, t_proj=10)
        for seed in (3, 4, 5):
            a = rp.replan(req, cfg, eng, mppi.DeviceNoise(seed), graph=True)
            b = rp.replan(req, cfg, eng, mppi.DeviceNoise(seed), graph=False)
            assert (a is None) == (b is None)
            if a is not None:
                np.testing.assert_array_equal(a.gains, b.gains)
                np.testing.assert_array_equal(a.nominal.inputs, b.nominal.inputs)
                np.testing.assert_array_equal(a.nominal.states, b.nominal.states)
                assert a.nominal.t_start == b.nominal.t_start
    plan = mppi.engine_plan(eng)
    assert len(plan._replan_graphs) == 2
    req = rp.ReplanRequest(x=x0, fluid=vpm.FluidState.empty(cfg.vpm), policy=pol, t=0.0, t_proj=10)
    ms = {}
    for g in (True, False):
        rp.replan(req, cfg, eng, mppi.DeviceNoise(1), graph=g)
        t0 = time.perf_counter()
        for i in range(5):
            rp.replan(req, cfg, eng, mppi.DeviceNoise(i), graph=g)
        ms[g] = 1e3 * (time.perf_counter() - t0) / 5
    print(f"replan e2e: graph {ms[True]:.3f} ms, eager {ms[False]:.3f} ms")


def test_bootstrap_with_device_noise(torch_cuda):
    """bootstrap_policy (annealed MPPI + nominal + build_policy) runs end to end with
    a DeviceNoise generator and is deterministic."""
    from paper_2509_16079_b200 import config, mppi, replan as rp, rollout
    cfg = config.ExperimentConfig()
    cfg.mppi.batch = 128
    cfg.scenario.bootstrap_iterations = 3
    eng = rollout.Engine.from_config(cfg)
    a = rp.bootstrap_policy(cfg, eng, mppi.DeviceNoise(2))
    b = rp.bootstrap_policy(cfg, eng, mppi.DeviceNoise(2))
    np.testing.assert_array_equal(a.gains, b.gains)
    np.testing.assert_array_equal(a.nominal.inputs, b.nominal.inputs)
    assert np.isfinite(a.gains).all()
