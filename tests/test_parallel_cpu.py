"""Multi-process (gloo, world_size 2 and 8) tests of the sharding logic, computed by the CPU oracle.

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


# ---------------------------------------------------------------------------------------------
# world 8 (the 8-GPU box), gloo on CPU: one spawned process per rank runs a named
# scenario; results come back through a queue keyed by rank.
def _scenario(rank, world, port, q, name, arg):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, SCENARIOS[name](rank, world, arg)))
    except Exception as e:  # noqa: BLE001 -- reported to the test
        q.put((rank, ("raised", type(e).__name__, str(e))))
    finally:
        dist.destroy_process_group()


def _channels(rank, world, n_channels):
    panel = synthetic.roi(synthetic.rayonix_panel(), 1900, 1890, 6, 10)
    ctx = synthetic.ls49_context(panel=panel, n_channels=n_channels, n_domains=2, compute="fp64")
    out = PixelBuffer.zeros(ctx.panel.dims, "f64")
    res = parallel.simulate_channel_sharded(ctx, out, partial=oracle_partial, finalize=host_finalize)
    return None if res is None else res.data.copy()


def _subgroup(rank, world, n_channels):
    """Ranks 1, 3, 5 form a group whose root is its member 1 (global rank 3)."""
    members = [1, 3, 5]
    group = dist.new_group(members)
    if rank not in members:
        return "outside"
    panel = synthetic.roi(synthetic.rayonix_panel(), 1900, 1890, 6, 10)
    ctx = synthetic.ls49_context(panel=panel, n_channels=n_channels, n_domains=2, compute="fp64")
    out = PixelBuffer.zeros(ctx.panel.dims, "f64")
    res = parallel.simulate_channel_sharded(ctx, out, group=group, root=1, partial=oracle_partial,
                                            finalize=host_finalize)
    return None if res is None else res.data.copy()


def _campaign_indices(rank, world, arg):
    from paper_2205_07976_b200.io import campaign_indices

    n_images, first = arg
    return campaign_indices(n_images, first)


SCENARIOS = {"channels": _channels, "subgroup": _subgroup, "campaign_indices": _campaign_indices}


def run_world(name, arg, world=8):
    ctxm = mp.get_context("spawn")
    q = ctxm.Queue()
    port = free_port()
    procs = [ctxm.Process(target=_scenario, args=(r, world, port, q, name, arg)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return [got[r] for r in range(world)]


@pytest.mark.parametrize("n_channels", [1000, 100, 13])
def test_channel_sharded_world8_uneven_shards(n_channels):
    """1000 / 100 / 13 channels over 8 ranks (shards of 125, 12-13 and 1-2 channels): the root's
    image equals the whole image; every other rank returns None."""
    from oracle import oracle

    panel = synthetic.roi(synthetic.rayonix_panel(), 1900, 1890, 6, 10)
    ctx = synthetic.ls49_context(panel=panel, n_channels=n_channels, n_domains=2, compute="fp64")
    want, _ = oracle.spots(describe(ctx), "f64", nthreads=4)
    got = run_world("channels", n_channels)
    assert all(g is None for g in got[1:]), got[1:]
    np.testing.assert_allclose(got[0], want, rtol=1e-13, atol=0)


def test_channel_sharded_world8_fewer_channels_than_ranks():
    """7 channels over 8 ranks: every rank raises the same ValueError (no rank blocks in a collective)."""
    got = run_world("channels", 7)
    assert all(g[0] == "raised" and g[1] == "ValueError" for g in got), got


def test_channel_sharded_subgroup_root_is_group_local():
    """root is a rank of the group: group [1, 3, 5] with root 1 delivers the image on global rank 3."""
    from oracle import oracle

    panel = synthetic.roi(synthetic.rayonix_panel(), 1900, 1890, 6, 10)
    ctx = synthetic.ls49_context(panel=panel, n_channels=9, n_domains=2, compute="fp64")
    want, _ = oracle.spots(describe(ctx), "f64", nthreads=4)
    got = run_world("subgroup", 9)
    assert [r for r in range(8) if isinstance(got[r], np.ndarray)] == [3]
    assert got[1] is None and got[5] is None and all(got[r] == "outside" for r in (0, 2, 4, 6, 7))
    np.testing.assert_allclose(got[3], want, rtol=1e-13, atol=0)


@pytest.mark.parametrize("n_images,first", [(1024, 0), (7, 3), (13, 100)])
def test_campaign_indices_world8_cover_once(n_images, first):
    """run_campaign's per-rank share at world 8 (C3: 1024 images over 8 GPUs): contiguous blocks in
    rank order, sizes within one, every image exactly once (scheduler.py:138-153)."""
    got = run_world("campaign_indices", (n_images, first))
    flat = [i for r in got for i in r]
    assert flat == list(range(first, first + n_images))
    sizes = [len(r) for r in got]
    assert max(sizes) - min(sizes) <= 1
