"""Multi-process (gloo, world_size 2) tests of the sharding logic, computed by the CPU oracle.

The GPU library is swapped for the oracle only HERE (test infrastructure):
the decomposition (shard ranges, global norm, reduce, root-side scale) is the
product code in paper_2205_07976_b200.parallel.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2205_07976_b200 import PixelBuffer, describe, parallel, synthetic


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def small_ctx():
    panel = synthetic.roi(synthetic.rayonix_panel(), 1900, 1890, 12, 20)
    return synthetic.ls49_context(panel=panel, n_channels=7, n_domains=2, compute="fp64")


def oracle_partial(ctx, lo, hi, norm):
    from oracle import oracle

    raw = np.zeros(ctx.panel.n_pixels)
    if hi > lo:
        oracle.spots(describe(ctx, src_begin=lo, src_end=hi, norm=norm), "raw", out=raw, nthreads=1)
    return torch.from_numpy(raw), oracle.scale(describe(ctx, norm=norm))


def host_finalize(raw, scale, out):
    vals = scale * raw.numpy()
    out.data[:] = vals.astype(out.data.dtype)


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ctx = small_ctx()
        out = PixelBuffer.zeros(ctx.panel.dims, "f64")
        res = parallel.simulate_channel_sharded(ctx, out, partial=oracle_partial, finalize=host_finalize)
        if rank == 0:
            q.put(res.data.copy())
        else:
            q.put(None if res is None else "non-root returned an image")
    finally:
        dist.destroy_process_group()


def test_plan_batches_partition():
    for n in (0, 1, 7, 1024):
        for r in (1, 2, 3, 8):
            b = parallel.plan_batches(n, r)
            sizes = [hi - lo for _, (lo, hi) in b]
            assert sum(sizes) == n and max(sizes) - min(sizes) <= 1
            assert [lo for _, (lo, _) in b] == sorted(lo for _, (lo, _) in b)
            cover = [i for _, (lo, hi) in b for i in range(lo, hi)]
            assert cover == list(range(n))


def test_global_norm_matches_descriptor_default():
    ctx = small_ctx()
    from oracle import oracle

    assert oracle.scale(describe(ctx)) == pytest.approx(oracle.scale(describe(ctx, norm=parallel.global_norm(ctx))),
                                                        rel=1e-15)


def test_channel_sharded_world2_equals_whole_image():
    ctx = small_ctx()
    from oracle import oracle

    want, _ = oracle.spots(describe(ctx), "f64", nthreads=2)
    ctxm = mp.get_context("spawn")
    q = ctxm.Queue()
    port = free_port()
    procs = [ctxm.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    img = next(g for g in got if isinstance(g, np.ndarray))
    assert sum(1 for g in got if g is None) == 1
    np.testing.assert_allclose(img, want, rtol=1e-13, atol=0)
