"""GPU: run_point's per-batch device counters and the multi-GPU sweep entry point
(one host thread per device, one NCCL int64 all-reduce) against single-device sums and
the compiled reference."""
import math

import numpy as np
import pytest

import oracle as O
import paper_1505_04979_b200 as P
from paper_1505_04979_b200.dist import COUNTER_FIELDS

pytestmark = pytest.mark.gpu
Z0 = math.exp(-0.5)
LIB = O.REF or O.C


@pytest.mark.parametrize("n,generic", [(1024, False), (4096, False), (16384, False), (1024, True)],
                         ids=["warp", "cta", "cluster", "generic"])
def test_simulate_batches_per_batch_counters(ctx, n, generic):
    code = P.PolarCode.construct(n, n // 2, Z0)
    frames = 1000 if n == 1024 else 600
    ctx.force_generic(generic)
    try:
        b = P.simulate_batches(code, "csfg", 2, 100, frames, 2.5, batch=256, ctx=ctx)
        whole = P.simulate_point(code, "csfg", 2, 100, frames, 2.5, ctx=ctx)
    finally:
        ctx.force_generic(False)
    nb = (frames + 255) // 256
    assert b.shape == (nb, 10)
    assert list(b[:, 0]) == [256] * (nb - 1) + [frames - 256 * (nb - 1)]
    assert [int(x) for x in b.sum(0)] == [whole[k] for k in COUNTER_FIELDS]
    # batch 1 (trials 356..611) against the reference compiled in fp32, frame by frame summed
    info, llr = O.trials(2, 356, 256, code.frozen, 2.5, lib=LIB)
    r = O.decode_batch("csfg", code.frozen, llr.astype(np.float32), prec=32, lib=LIB)
    be = (r["u_hat"][:, code.frozen == 0] != info).sum(1)
    it = r["iterations"].astype(np.int64)
    exp = [256, be.sum(), (be > 0).sum(), it.sum(), (it * it).sum(), r["pe"].sum(), r["n_events"].sum(),
           (r["stop"] == 0).sum(), (r["stop"] == 1).sum(), (r["stop"] == 2).sum()]
    assert [int(x) for x in b[1]] == [int(x) for x in exp]


def test_sweep_multi_equals_single_device_sums():
    """pbp_simulate_sweep_multi on the visible devices (NCCL all-reduce; one device on the
    test box) equals the per-point single-context counters."""
    code = P.PolarCode.construct(1024, 512, Z0)
    snrs = [2.0, 3.0]
    got = P.simulate_sweep_multi(code, "csfg", 2, 3000, snrs)
    ctx = P.Context(0)
    for snr, row in zip(snrs, got):
        assert row == P.simulate_point(code, "csfg", 2, 0, 3000, snr, ctx=ctx)


def test_sweep_multi_rejects_bad_arguments():
    code = P.PolarCode.construct(256, 128, Z0)
    with pytest.raises(ValueError):
        P.simulate_sweep_multi(code, "csfg", 2, 100, [], devices=[0])
    with pytest.raises(ValueError):
        P.simulate_sweep_multi(code, "csfg", 2, -1, [1.0], devices=[0])


def test_run_point_stop_rule_matches_batchwise_oracle(ctx):
    """The 256-frame stop rule of run_point on device batch counters: the point stops on the
    first batch boundary where every decoder has min_frame_errors, as the reference."""
    code = P.PolarCode.construct(256, 128, Z0)
    cfg = P.SimConfig(code=code, decoders=(1, 2), min_frame_errors=40, max_frames=20_000, seed=7)
    rows = P.run_point(cfg, 1.5, ctx=ctx)
    frames = rows[0].frames
    assert frames % 256 == 0 and all(r.frames == frames for r in rows)
    info, llr = O.trials(7, 0, frames, code.frozen, 1.5, lib=LIB)
    fe = {}
    for kind in ("gmatrix", "csfg"):
        r = O.decode_batch(kind, code.frozen, llr.astype(np.float32), prec=32, lib=LIB)
        err = ((r["u_hat"][:, code.frozen == 0] != info).sum(1) > 0).astype(np.int64)
        fe[kind] = np.cumsum(err)
    stop = next(b for b in range(256, frames + 1, 256)
                if fe["gmatrix"][b - 1] >= 40 and fe["csfg"][b - 1] >= 40)
    assert stop == frames
    assert rows[0].frame_errors == fe["gmatrix"][-1] and rows[1].frame_errors == fe["csfg"][-1]


@pytest.mark.parametrize("n", [1024, 4096])
def test_decode_count_batches_one_launch_per_sweep(ctx, n):
    """pbp_decode_count_batches_device over a sweep stored point after point (bench.py's
    timed launch): one counter set per point, equal to each point's simulate_point."""
    import ctypes as C
    import torch
    code = P.PolarCode.construct(n, n // 2, Z0)
    snrs, frames = [1.5, 2.5, 3.5], 700 if n == 1024 else 300
    llr = np.concatenate([P.generate(code, 2, 50, frames, s, ctx=ctx)[0] for s in snrs])
    u = np.concatenate([P.generate(code, 2, 50, frames, s, ctx=ctx)[1] for s in snrs])
    dev = torch.device("cuda", ctx.device)
    d_llr = torch.from_numpy(llr).to(dev)
    d_u = torch.from_numpy(u.view(np.int32)).to(dev)
    cnt = torch.zeros((len(snrs), 10), dtype=torch.int64, device=dev)
    cs = code.c_struct()
    torch.cuda.synchronize(dev)
    P._check(P.lib.pbp_decode_count_batches_device(ctx.handle, C.byref(cs), 2, P._abi.f32p(d_llr.data_ptr()),
                                                   P._abi.u32p(d_u.data_ptr()), len(snrs) * frames, frames,
                                                   0.9375, 40, P._abi.i64p(cnt.data_ptr()), None))
    ctx.synchronize()
    got = cnt.cpu().numpy()
    for i, s in enumerate(snrs):
        want = P.simulate_point(code, "csfg", 2, 50, frames, s, ctx=ctx)
        assert [int(x) for x in got[i]] == [want[k] for k in COUNTER_FIELDS]
    with pytest.raises(ValueError):
        P._check(P.lib.pbp_decode_count_batches_device(ctx.handle, C.byref(cs), 2, P._abi.f32p(d_llr.data_ptr()),
                                                       P._abi.u32p(d_u.data_ptr()), frames, 0, 0.9375, 40,
                                                       P._abi.i64p(cnt.data_ptr()), None))


def _gloo_gpu_worker(rank, world, port, q):
    import os
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch.distributed as dist
    import paper_1505_04979_b200 as P
    from paper_1505_04979_b200 import dist as D
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    pctx = P.Context(0)  # one GPU on the test box: both ranks decode their shards on it

    def gpu_point(code, decoder, seed, first, count, ebn0, alpha, max_iter):
        return P.simulate_point(code, decoder, seed, first, count, ebn0, alpha, max_iter, ctx=pctx)

    out = []
    for n, frames, snrs in ((1024, 2001, [2.0, 3.5]), (16384, 151, [2.5])):
        code = P.PolarCode.construct(n, n // 2, Z0)
        out.append(D.simulate_sweep_sharded(code, "csfg", 5, frames, snrs, rank=rank, world=world,
                                            point_fn=gpu_point))
    q.put((rank, out))
    dist.destroy_process_group()


@pytest.mark.timeout(600, method="thread")
def test_gloo_world2_gpu_shards_equal_single_process():
    """dist.simulate_sweep_sharded with the GPU decoder per rank (gloo world of 2; the
    counters all-reduced on the host): the sums equal one process decoding every trial,
    at n = 1024 (warp kernel) and n = 16384 (2-CTA cluster kernel)."""
    import socket

    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    mctx = mp.get_context("spawn")
    q = mctx.Queue()
    procs = [mctx.Process(target=_gloo_gpu_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=500) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[0] == res[1]
    ctx = P.Context(0)
    for (n, frames, snrs), got in zip(((1024, 2001, [2.0, 3.5]), (16384, 151, [2.5])), res[0]):
        code = P.PolarCode.construct(n, n // 2, Z0)
        whole = [P.simulate_point(code, "csfg", 5, 0, frames, snr, ctx=ctx) for snr in snrs]
        assert got == whole, n
