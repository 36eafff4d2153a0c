"""Multi-GPU partitioning of the spot path.

One process per GPU (torchrun), torch.distributed for the plumbing.

* Image sharding (config C3): independent images, contiguous index blocks
  whose sizes differ by at most one (the reference's plan_batches,
  scheduler.py:138-153).  No data-path collective; images are bit-identical
  to a 1-GPU run.
* Channel sharding (config C5, one huge image): rank g evaluates sources
  [c_g, c_{g+1}) into an UNSCALED FP64 partial image with the GLOBAL
  normalisation (kernels.py:243-245); one reduce(SUM) to the root over
  NCCL/NVLink, and the root applies r_e^2 fluence / norm and stores
  (nbx_finalize).  Summation order differs from 1 GPU, so the result agrees
  to rounding, not bitwise.

The compute of a partial and the finalize step are injectable so the
decomposition logic can be tested with gloo on CPU against the oracle; the
defaults are the GPU library and there is no CPU fallback.
"""
from __future__ import annotations

from typing import Callable


from .kernels import PixelBuffer, SpotsContext, SpotsPlan
from . import _native as N

__all__ = ["plan_batches", "channel_shards", "global_norm", "shard_images", "simulate_channel_sharded"]


def plan_batches(n_images: int, ranks: int) -> list[tuple[int, tuple[int, int]]]:
    """Contiguous partition of [0, n_images) over ranks; the first n % ranks take one extra."""
    if ranks < 1:
        raise ValueError("ranks must be >= 1")
    if n_images < 0:
        raise ValueError("n_images must be >= 0")
    base, extra = divmod(n_images, ranks)
    out, start = [], 0
    for r in range(ranks):
        size = base + (1 if r < extra else 0)
        out.append((r, (start, start + size)))
        start += size
    return out


def channel_shards(n_sources: int, ranks: int) -> list[tuple[int, int]]:
    """[begin, end) source ranges per rank, balanced to within one channel."""
    return [rng for _, rng in plan_batches(n_sources, ranks)]


def global_norm(ctx: SpotsContext) -> float:
    """sum(weights) * n_domains * oversample^2 over the WHOLE spectrum (kernels.py:243-245)."""
    phi = getattr(ctx, "phi", None)
    n_dom = len(ctx.crystal.mosaic) * (phi.steps if phi is not None else 1)
    return float(ctx.spectrum.weights.sum()) * n_dom * ctx.oversample * ctx.oversample


def shard_images(n_images: int, rank: int, world: int) -> range:
    _, (lo, hi) = plan_batches(n_images, world)[rank]
    return range(lo, hi)


def _gpu_partial(ctx: SpotsContext, lo: int, hi: int, norm: float):
    """Unscaled FP64 partial of sources [lo, hi) in a CUDA tensor (+ the plan's global scale)."""
    import torch

    plan = SpotsPlan(ctx, src_begin=lo, src_end=hi, norm=norm, device=torch.cuda.current_device())
    raw = torch.zeros(plan.n_pixels, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    if hi > lo:
        plan.run(raw.data_ptr(), mode=N.OUT_RAW_F64, on_device=True)
    scale = plan.scale
    plan.close()
    return raw, scale


def _gpu_finalize(raw, scale: float, out: PixelBuffer):
    cx = N.context(raw.device.index)
    mode = N.OUT_F32 if out.precision == "f32" else N.OUT_F64
    bad = N.C.c_int64(-1)
    with cx.lock:
        status = cx.lib.nbx_finalize(cx.handle, raw.data_ptr(), raw.numel(), scale, mode, out.data.ctypes.data, 0,
                                     N.C.byref(bad))
        N.check(cx, status, bad.value)


def _p2p_channel_sharded(ctx: SpotsContext, out: PixelBuffer | None, group, root: int, world: int, rank: int):
    """Fused transport: every rank's spot kernel stores its FP64 partial straight into its slot of
    an IPC-shared buffer on the root (NBX_OUT_RAW_STORE_F64 epilogue, the transfer overlapping
    the computation pixel by pixel); after a barrier the root sums the slots in rank order."""
    import torch
    import torch.distributed as dist

    dev = torch.cuda.current_device()
    cx = N.context(dev)
    lo, hi = channel_shards(len(ctx.spectrum.samples), world)[rank]
    plan = SpotsPlan(ctx, src_begin=lo, src_end=hi, norm=global_norm(ctx), device=dev)
    npix = plan.n_pixels
    base = N.C.c_void_p()
    handle = [None]
    if rank == root:
        buf = N.C.create_string_buffer(64)
        with cx.lock:
            N.check(cx, cx.lib.nbx_ipc_alloc(cx.handle, world * npix * 8, N.C.byref(base), buf))
        handle = [bytes(buf.raw)]
    dist.broadcast_object_list(handle, src=root, group=group)
    if rank != root:
        with cx.lock:
            N.check(cx, cx.lib.nbx_ipc_open(cx.handle, handle[0], N.C.byref(base)))
    try:
        slot = base.value + rank * npix * 8
        torch.cuda.synchronize()
        plan.run(slot, mode=N.OUT_RAW_STORE_F64, on_device=True)  # synchronous: our stores are done
        scale = plan.scale
        dist.barrier(group=group)  # every rank's slot is written
        result = None
        if rank == root:
            result = out if out is not None else PixelBuffer.zeros(ctx.panel.dims, "f32")
            mode = N.OUT_F32 if result.precision == "f32" else N.OUT_F64
            bad = N.C.c_int64(-1)
            with cx.lock:
                st = cx.lib.nbx_reduce_slots(cx.handle, base.value, world, npix, scale, mode,
                                             result.data.ctypes.data, 0, N.C.byref(bad))
                N.check(cx, st, bad.value)
        dist.barrier(group=group)  # the root has read every slot
    finally:
        plan.close()
        with cx.lock:
            if rank == root:
                cx.lib.nbx_ipc_free(cx.handle, base)
            else:
                cx.lib.nbx_ipc_close(cx.handle, base)
    return result


def simulate_channel_sharded(ctx: SpotsContext, out: PixelBuffer | None = None, *, group=None, root: int = 0,
                             partial: Callable | None = None, finalize: Callable | None = None,
                             transport: str = "nccl"):
    """One image split by energy channel over the ranks of ``group``; returns the image on root, else None.

    ``transport="nccl"`` (default, the north star's NCCL reduce): partial images in CUDA
    tensors, one ``dist.reduce`` to the root, scale + store there.  ``transport="p2p"``: the
    partials are stored by each rank's kernel directly into the root's memory (CUDA IPC /
    NVLink peer stores) and summed there in rank order -- no separate collective.
    ``partial(ctx, lo, hi, norm) -> (raw_tensor, scale)`` and ``finalize(raw_tensor, scale,
    out)`` (NCCL transport) default to the GPU library.
    """
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    if transport == "p2p" and world > 1:
        if len(ctx.spectrum.samples) < world:
            raise ValueError(f"{len(ctx.spectrum.samples)} sources cannot be split over {world} ranks")
        return _p2p_channel_sharded(ctx, out, group, root, world, rank)
    if transport not in ("nccl", "p2p"):
        raise ValueError("transport must be 'nccl' or 'p2p'")
    partial = partial or _gpu_partial
    finalize = finalize or _gpu_finalize
    n_src = len(ctx.spectrum.samples)
    if n_src < world:
        raise ValueError(f"{n_src} sources cannot be split over {world} ranks")
    lo, hi = channel_shards(n_src, world)[rank]
    raw, scale = partial(ctx, lo, hi, global_norm(ctx))
    if world > 1:
        dist.reduce(raw, dst=root, op=dist.ReduceOp.SUM, group=group)
    if rank != root:
        return None
    if out is None:
        out = PixelBuffer.zeros(ctx.panel.dims, "f32")
    finalize(raw, scale, out)
    return out
