"""CPU: the multi-GPU host path (trial sharding + one int64 all-reduce) on a gloo
world of size 2. The per-shard counters come from the oracle here (no GPU in the
CPU suite); on the B200 box the same function runs the GPU decoder per rank."""
import math
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1505_04979_b200 import dist as D

Z0 = math.exp(-0.5)


def oracle_point(code, decoder, seed, first, count, ebn0, alpha, max_iter):
    import oracle as O
    info, llr = O.trials(seed, first, count, code.frozen, ebn0, lib=O.C)
    r = O.decode_batch(decoder, code.frozen, llr.astype(np.float32), alpha, max_iter, prec=32, threads=2)
    be = (r["u_hat"][:, code.frozen == 0] != info).sum(1)
    it = r["iterations"].astype(np.int64)
    return {"frames": count, "bit_errors": int(be.sum()), "frame_errors": int((be > 0).sum()),
            "sum_iters": int(it.sum()), "sum_iters_sq": int((it * it).sum()), "sum_pe": int(r["pe"].sum()),
            "sum_events": int(r["n_events"].sum()),
            "stop_max_iter": int((r["stop"] == 0).sum()), "stop_gmatrix": int((r["stop"] == 1).sum()),
            "stop_csfg": int((r["stop"] == 2).sum())}


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch.distributed as dist
    import paper_1505_04979_b200 as P
    from paper_1505_04979_b200 import dist as D2
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    code = P.PolarCode.construct(64, 32, Z0)
    out = D2.simulate_sweep_sharded(code, "csfg", 7, 101, [1.5, 3.0], rank=rank, world=world,
                                    point_fn=oracle_point)
    q.put((rank, out))
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_shard_range_partitions():
    for total in (0, 1, 7, 100, 100001):
        for world in (1, 2, 3, 8):
            spans = [D.shard_range(total, r, world) for r in range(world)]
            assert spans[0][0] == 0
            assert sum(c for _, c in spans) == total
            for (f0, c0), (f1, _) in zip(spans, spans[1:]):
                assert f0 + c0 == f1
    with pytest.raises(ValueError):
        D.shard_range(10, 2, 2)


def test_gloo_world2_sharded_counters_equal_single_process():
    import paper_1505_04979_b200 as P
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[0] == res[1]  # every rank holds the reduced sums
    code = P.PolarCode.construct(64, 32, Z0)
    whole = [oracle_point(code, "csfg", 7, 0, 101, snr, 0.9375, 40) for snr in (1.5, 3.0)]
    assert res[0] == whole
