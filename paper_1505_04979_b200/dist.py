"""Multi-GPU Monte-Carlo: shard trial ranges across ranks, combine counters once.

SURVEY.md 8(e): a trial depends only on (seed, trial) (src/sim_harness.cpp:67) and no
state crosses frames, so rank r of W decodes the contiguous trial range
[r*F/W, (r+1)*F/W) on its own GPU and the Accumulator fields (src/sim_harness.cpp:56-63,
plus the event count and stop-reason histogram) are summed with ONE int64 all-reduce
(NCCL over NVLink / NVSwitch on the B200 box; gloo in the CPU tests). Integer sums make
the result identical to the single-GPU and CPU aggregates for any world size.

One process per GPU, launched by torchrun; nothing here runs kernels itself.
"""
from __future__ import annotations

from typing import Callable, Dict, Optional, Sequence

COUNTER_FIELDS = ("frames", "bit_errors", "frame_errors", "sum_iters", "sum_iters_sq", "sum_pe",
                  "sum_events", "stop_max_iter", "stop_gmatrix", "stop_csfg")


def shard_range(total: int, rank: int, world: int):
    """Contiguous trial range of `rank`: [first, first + count)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("shard_range: bad rank/world")
    if total < 0:
        raise ValueError("shard_range: total < 0")
    first = total * rank // world
    last = total * (rank + 1) // world
    return first, last - first


def allreduce_counters(per_point: Sequence[Dict[str, int]], group=None, device=None):
    """Sum a list of counter dicts over all ranks with one int64 all_reduce."""
    import torch
    import torch.distributed as dist

    t = torch.tensor([[int(c[k]) for k in COUNTER_FIELDS] for c in per_point], dtype=torch.int64,
                     device=device)
    if dist.is_available() and dist.is_initialized():
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return [dict(zip(COUNTER_FIELDS, map(int, row))) for row in t.tolist()]


def simulate_sweep_sharded(code, decoder, seed: int, frames_per_point: int, snrs: Sequence[float],
                           alpha: float = 0.9375, max_iter: int = 40, rank: int = 0, world: int = 1,
                           group=None, device=None,
                           point_fn: Optional[Callable] = None):
    """run_sweep's counters with fixed frame counts (min_frame_errors = inf), sharded.

    point_fn(code, decoder, seed, first, count, ebn0, alpha, max_iter) -> counters dict;
    defaults to the GPU path (paper_1505_04979_b200.simulate_point on a Context of this
    rank's device: `device`, else LOCAL_RANK).
    Trial indices restart at 0 for every Eb/N0 point, as in run_point
    (src/sim_harness.cpp:141-147), so every point is sharded the same way.
    """
    if point_fn is None:
        import os

        import paper_1505_04979_b200 as P
        # this rank's GPU: the `device` argument, else torchrun's LOCAL_RANK
        dev = device if device is not None else int(os.environ.get("LOCAL_RANK", "0"))
        dev = dev.index if hasattr(dev, "index") and dev.index is not None else int(dev)
        pctx = P.Context(dev)

        def point_fn(code, decoder, seed, first, count, ebn0, alpha, max_iter):
            return P.simulate_point(code, decoder, seed, first, count, ebn0, alpha, max_iter, ctx=pctx)
    first, count = shard_range(frames_per_point, rank, world)
    local = [point_fn(code, decoder, seed, first, count, snr, alpha, max_iter) for snr in snrs]
    return allreduce_counters(local, group=group, device=device)
