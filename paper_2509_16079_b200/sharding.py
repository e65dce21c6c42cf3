"""Multi-GPU MPPI: rollout rows sharded across ranks, one collective per iteration.

One process per GPU (``torch.distributed``, NCCL over NVLink).  The B = K+1
candidate rows (row 0 = incumbent) are split into contiguous blocks
(:func:`row_range`); every rank forks the same replicated fluid snapshot and u*
and runs only its rows.  The softmax update of mppi.py:46-59 is split exactly:

    rank r:  J_min_r,  Z_r = sum_b exp(-(J_b - J_min_r)/lambda),  S_r = sum_b w_b u_b
    gather:  one all_gather of W x (H+2) float64
    every rank:  J_min = min_r J_min_r,  u* = sum_r e_r S_r / sum_r e_r Z_r,
                 e_r = exp(-(J_min_r - J_min)/lambda), summed in rank order

so all ranks hold a bitwise-identical u* after every iteration with no other
traffic.  The partial and combine run as device kernels (``vpm_mppi_partial`` /
``vpm_mppi_combine``); only the gather is a collective.
"""

from __future__ import annotations


def row_range(B: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous block of rows [begin, end) owned by ``rank``; sizes differ by <= 1
    and rank 0 owns the incumbent row 0."""
    base, extra = divmod(B, world)
    begin = rank * base + min(rank, extra)
    return begin, begin + base + (1 if rank < extra else 0)


def gather_partials(partial, group=None):
    """All-gather every rank's (H+2) partial into a (W, H+2) tensor in rank order.
    Device-agnostic: NCCL for CUDA tensors, gloo for CPU tensors (tests)."""
    import torch
    import torch.distributed as dist
    W = dist.get_world_size(group)
    flat = partial.contiguous().view(-1)
    out = torch.empty((W, flat.numel()), dtype=partial.dtype, device=partial.device)
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(out, flat, group=group)   # one NCCL all-gather
    elif flat.is_cuda:
        # gloo has no all_gather for CUDA tensors: gather through host memory
        # (functional multi-process tests on one device; 416 bytes per rank)
        host = flat.cpu()
        parts = [torch.empty_like(host) for _ in range(W)]
        dist.all_gather(parts, host, group=group)
        out.copy_(torch.stack(parts))
    else:
        dist.all_gather(list(out.unbind(0)), flat, group=group)
    return out


class ShardedMppi:
    """Device-resident MPPI over ``world`` ranks (``world == 1`` skips the gather).

    Holds the plan, the replicated snapshot/u*, this rank's noise rows and all
    scratch, so an iteration allocates nothing.
    """

    def __init__(self, plan, x0, warm, noise_rows, *, B: int, sigma: float, temperature: float,
                 q, x_perch, rank: int = 0, world: int = 1, group=None):
        import torch
        self.torch = torch
        self.plan = plan
        self.B, self.sigma, self.temperature = int(B), float(sigma), float(temperature)
        self.rank, self.world, self.group = rank, world, group
        self.begin, self.end = row_range(self.B, world, rank)
        dev = x0.device
        self.x0 = x0
        self.ustar = warm.clone()
        self.T = int(warm.shape[0])
        self.q, self.xp = q, x_perch
        # noise_rows: (B-1, T) global noise; the kernel indexes it by global row
        self.noise = noise_rows
        rows = self.end - self.begin
        f64 = dict(dtype=torch.float64, device=dev)
        self.out = {"status": torch.empty(rows, dtype=torch.int64, device=dev),
                    "finals": torch.empty(rows, 7, **f64), "cost": torch.empty(rows, **f64)}
        self.partial = torch.empty(self.T + 2, **f64)
        self.flag = torch.zeros(1, dtype=torch.int32, device=dev)

    def reset(self) -> None:
        """Start a new optimisation: clear the sticky all-candidates-failed flag."""
        self.flag.zero_()

    def set_noise(self, noise_rows):
        self.noise = noise_rows

    def draw_noise(self, seed: int, iteration: int, stream=None):
        """Performance mode: draw this rank's noise rows on the device (Philox keyed
        by (seed, iteration, global row), so the union over ranks is the same matrix
        for any world size) into the global-row-indexed noise buffer."""
        from .device import noise_philox
        lo, hi = max(self.begin - 1, 0), self.end - 1  # noise row of global row g is g - 1
        if hi > lo:
            noise_philox(seed, iteration, self.noise[lo:hi], row_begin=lo, stream=stream)

    def iteration(self, stream=None) -> None:
        from .device import mppi_combine
        rows = self.end - self.begin
        self.plan.batch(self.x0, self.T, ustar=self.ustar, noise=self.noise, sigma=self.sigma,
                        row_begin=self.begin, rows=rows, q=self.q, x_perch=self.xp, out=self.out,
                        stream=stream)
        self.plan.mppi_partial(self.out["cost"], self.ustar, self.noise, self.sigma,
                               self.temperature, row_begin=self.begin, partial=self.partial,
                               stream=stream)
        # world 1 without an explicit group: no collective at all; with a group (any
        # size, e.g. a world-1 NCCL group in tests) the partials go through it
        if self.world == 1 and self.group is None:
            parts = self.partial.view(1, -1)
        else:
            parts = gather_partials(self.partial, self.group)
        mppi_combine(parts, self.temperature, self.ustar, self.flag, stream=stream)

    def check(self) -> None:
        """Raise like mppi.py:55-56 if any iteration since the last reset() had every
        candidate fail (the combine kernel's flag is sticky; a later successful
        iteration does not clear it)."""
        if int(self.flag.item()) != 0:
            raise ValueError("all sampled rollouts failed (infinite cost)")

    kernels_per_iteration = 3

