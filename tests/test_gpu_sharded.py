"""Sharded MPPI on the device (paper_2509_16079_b200/sharding.py).

gpurun offers one GPU, so the rank protocol is exercised two ways on cuda:0:
  * in-process shards: W row blocks (W = 2, 3, 8) run as separate launches, their
    device partials stacked in rank order and combined -- per-row results must be
    bitwise identical to the single-shard launch (rows do not depend on the launch
    they are part of) and u* must match the single-shard u* to FP64 rounding of
    the per-shard rescaling (rtol 1e-12);
  * a real 2-process run (torch.distributed, gloo through host memory instead of
    NCCL, both ranks on cuda:0): both ranks end with a bitwise-identical u* equal
    to the in-process W = 2 result.  The ranks' kernels never wait on each other.
"""
import os
import socket

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu

K, H, SIGMA, LAM = 1024, 50, 2.0, 0.05
Q = [10, 10, 1, 0, 0.2, 0.2, 0.2]
XP = [3.5, 0, np.pi / 4, 0, 0.5, -0.5, 0]


def _setup(torch, dev):
    from paper_2509_16079_b200.device import DevicePlan
    sc = golden("scenario_C4.npz")
    flat = (sc["wake_pos"], sc["wake_gamma"], sc["wake_age"], int(sc["n_wake"]), int(sc["ring_a"]),
            int(sc["ring_b"]), sc["prev_pos"], sc["prev_gamma"], int(sc["n_prev"]),
            float(sc["prev_lev"]), sc["ema"])
    plan = DevicePlan(sc["iparams"], sc["fparams"], device=dev.index or 0)
    plan.set_fluid(flat)
    f64 = lambda a: torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64), device=dev)
    noise = f64(np.random.default_rng(21).normal(0.0, 1.0, (K, H)))
    return plan, f64(sc["x0"]), f64(np.full(H, -6.0)), noise, f64(Q), f64(XP)


def _sharded_ustar(torch, plan, x0, warm, noise, q, xp, W):
    """Rank-by-rank emulation of ShardedMppi.iteration in one process."""
    from paper_2509_16079_b200.device import mppi_combine
    from paper_2509_16079_b200.sharding import row_range
    parts, costs = [], []
    for r in range(W):
        b, e = row_range(K + 1, W, r)
        o = plan.batch(x0, H, ustar=warm, noise=noise, sigma=SIGMA, row_begin=b, rows=e - b, q=q,
                       x_perch=xp)
        parts.append(plan.mppi_partial(o["cost"], warm, noise, SIGMA, LAM, row_begin=b))
        costs.append(o["cost"])
    u = warm.clone()
    flag = torch.zeros(1, dtype=torch.int32, device=warm.device)
    mppi_combine(torch.stack(parts), LAM, u, flag)
    torch.cuda.synchronize()
    assert int(flag.item()) == 0
    return u.cpu().numpy(), torch.cat(costs).cpu().numpy()


def test_in_process_shards_match_single_launch():
    import torch
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    plan, x0, warm, noise, q, xp = _setup(torch, dev)
    u1, c1 = _sharded_ustar(torch, plan, x0, warm, noise, q, xp, 1)
    for W in (2, 3, 8):
        uw, cw = _sharded_ustar(torch, plan, x0, warm, noise, q, xp, W)
        np.testing.assert_array_equal(cw, c1)            # rows are launch-independent
        np.testing.assert_allclose(uw, u1, rtol=1e-12, atol=1e-13)
    assert not np.array_equal(u1, warm.cpu().numpy())


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank(rank, world, port, out_q):
    try:
        import sys
        import torch
        import torch.distributed as dist
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_2509_16079_b200.sharding import ShardedMppi
        dev = torch.device("cuda", 0)
        plan, x0, warm, noise, q, xp = _setup(torch, dev)
        mp_ = ShardedMppi(plan, x0, warm, noise, B=K + 1, sigma=SIGMA, temperature=LAM, q=q,
                          x_perch=xp, rank=rank, world=world)
        mp_.iteration()
        torch.cuda.synchronize()
        mp_.check()
        out_q.put((rank, mp_.ustar.cpu().numpy()))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as err:  # report instead of hanging the parent
        out_q.put((rank, repr(err)))


def test_two_process_ranks_agree():
    import torch
    import torch.multiprocessing as mp
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
    for r in range(world):
        assert not isinstance(res[r], str), res[r]
    assert np.array_equal(res[0], res[1])
    torch.cuda.set_device(0)
    plan, x0, warm, noise, qq, xp = _setup(torch, torch.device("cuda", 0))
    u2, _ = _sharded_ustar(torch, plan, x0, warm, noise, qq, xp, 2)
    np.testing.assert_array_equal(res[0], u2)


def test_failure_flag_is_sticky():
    """An all-candidates-failed iteration is not masked by a later successful one
    (ADVICE r1): check() raises until reset()."""
    import torch
    from paper_2509_16079_b200.sharding import ShardedMppi
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    plan, x0, warm, noise, q, xp = _setup(torch, dev)
    bad = x0.clone()
    bad[6] = 400.0  # leaves the envelope on the first step: every candidate fails
    mp_ = ShardedMppi(plan, bad, warm, noise, B=K + 1, sigma=SIGMA, temperature=LAM, q=q, x_perch=xp)
    mp_.iteration()
    mp_.x0 = x0
    mp_.iteration()
    torch.cuda.synchronize()
    with pytest.raises(ValueError):
        mp_.check()
    mp_.reset()
    mp_.iteration()
    mp_.check()


def _nccl_rank(port, out_q):
    try:
        import sys
        import torch
        import torch.distributed as dist
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), NCCL_DEBUG="INFO")
        torch.cuda.set_device(0)
        dev = torch.device("cuda", 0)
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
        from paper_2509_16079_b200.sharding import ShardedMppi
        plan, x0, warm, noise, q, xp = _setup(torch, dev)
        mp_ = ShardedMppi(plan, x0, warm, noise, B=K + 1, sigma=SIGMA, temperature=LAM, q=q, x_perch=xp,
                          rank=0, world=1, group=dist.group.WORLD)
        assert dist.get_backend(mp_.group) == "nccl"
        mp_.iteration()  # rollouts + partial + NCCL all_gather_into_tensor + combine
        torch.cuda.synchronize()
        mp_.check()
        out_q.put(("ok", mp_.ustar.cpu().numpy(), torch.cuda.nccl.version()))
        dist.destroy_process_group()
    except Exception as err:
        out_q.put(("err", repr(err), None))


def test_nccl_world1_all_gather_path():
    """The NCCL branch of gather_partials (all_gather_into_tensor) executed: a world-1
    NCCL process group on cuda:0 runs ShardedMppi.iteration through the collective;
    u* equals the no-collective single-GPU iteration bitwise."""
    import torch
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_nccl_rank, args=(_free_port(), q))
    p.start()
    status, u, ver = q.get(timeout=300)
    p.join(timeout=120)
    assert status == "ok", u
    print("NCCL", ver)
    torch.cuda.set_device(0)
    plan, x0, warm, noise, qq, xp = _setup(torch, torch.device("cuda", 0))
    u1, _ = _sharded_ustar(torch, plan, x0, warm, noise, qq, xp, 1)
    np.testing.assert_array_equal(u, u1)
