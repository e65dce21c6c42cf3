"""Multi-rank MPPI host logic on CPU: world_size-2 gloo processes run the same
partition / all-gather / rank-ordered combine protocol the NCCL path uses
(paper_2509_16079_b200/sharding.py), with the shard partials computed by the oracle."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def test_row_range_partitions_contiguously():
    from paper_2509_16079_b200.sharding import row_range
    for B in (1, 7, 257, 4097):
        for W in (1, 2, 3, 8):
            spans = [row_range(B, W, r) for r in range(W)]
            assert spans[0][0] == 0 and spans[-1][1] == B
            assert all(spans[i][1] == spans[i + 1][0] for i in range(W - 1))
            sizes = [e - b for b, e in spans]
            assert max(sizes) - min(sizes) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, J, cand, temp, out_q):
    try:
        import sys
        import torch
        import torch.distributed as dist
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from oracle import planner
        from paper_2509_16079_b200.sharding import gather_partials, row_range
        b, e = row_range(len(J), world, rank)
        part = torch.tensor(planner.shard_partial(J[b:e], cand[b:e], temp), dtype=torch.float64)
        gathered = gather_partials(part)
        u = planner.combine_partials(gathered.numpy(), temp)
        out_q.put((rank, u))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as err:  # report instead of hanging the parent
        out_q.put((rank, repr(err)))


@pytest.mark.parametrize("world", [2])
def test_sharded_update_matches_unsharded(world):
    from oracle import planner
    rng = np.random.default_rng(0)
    B, H, temp = 257, 50, 0.05
    J = rng.uniform(0.0, 3.0, B)
    J[rng.choice(B, 20, replace=False)] = np.inf          # failed rollouts
    J[200] = J.min() - 0.01                              # optimum in the last shard
    cand = rng.normal(-6.0, 2.0, (B, H))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, J, cand, temp, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ref = planner.weighted_mean(cand, J, temp)
    for r in range(world):
        np.testing.assert_allclose(res[r], ref, rtol=1e-12, atol=1e-12)
    assert np.array_equal(res[0], res[1])  # every rank holds the same u*
