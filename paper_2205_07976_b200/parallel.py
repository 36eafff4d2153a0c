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


def _global_rank(group, rank: int) -> int:
    """torch.distributed addresses src/dst by GLOBAL rank; ``root`` here is group-local."""
    import torch.distributed as dist

    return rank if group is None else dist.get_global_rank(group, rank)


def _all_ok(ok: bool, group) -> bool:
    """Every rank of ``group`` agrees whether all of them succeeded (MIN all-reduce of a flag)."""
    import torch
    import torch.distributed as dist

    dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
    flag = torch.tensor([1 if ok else 0], dtype=torch.int32, device=dev)
    dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=group)
    return bool(flag.item())


def _p2p_channel_sharded(ctx: SpotsContext, out: PixelBuffer | None, group, root: int, world: int, rank: int):
    """Fused transport: every rank's spot kernel stores its FP64 partial straight into its slot of
    an IPC-shared buffer on the root (NBX_OUT_RAW_STORE_F64 epilogue, the transfer overlapping
    the computation pixel by pixel); after a barrier the root sums the slots in rank order.

    Failure handling: each phase that can fail on one rank (plan build and slot allocation, slot
    mapping and the partial's kernel, the root's reduction) ends with an all-rank agreement on
    success, so no rank leaves a collective early and the root never frees the slots while a
    peer could still be storing into them; every rank then raises (its own error, or a
    RuntimeError naming the failed phase).
    """
    import torch
    import torch.distributed as dist

    dev = torch.cuda.current_device()
    cx = N.context(dev)
    groot = _global_rank(group, root)
    lo, hi = channel_shards(len(ctx.spectrum.samples), world)[rank]
    plan, base, handle, mapped, err = None, N.C.c_void_p(), [None], False, None
    try:  # phase 1: plan, and the root's slots
        plan = SpotsPlan(ctx, src_begin=lo, src_end=hi, norm=global_norm(ctx), device=dev)
        if rank == root:
            buf = N.C.create_string_buffer(64)
            with cx.lock:
                N.check(cx, cx.lib.nbx_ipc_alloc(cx.handle, world * plan.n_pixels * 8, N.C.byref(base), buf))
            mapped = True
            handle = [bytes(buf.raw)]
    except Exception as e:  # noqa: BLE001 -- re-raised after the ranks agree
        err = e
    result = None
    try:
        if not _all_ok(err is None, group):
            raise err or RuntimeError("channel shard set-up failed on another rank")
        dist.broadcast_object_list(handle, src=groot, group=group)
        npix = plan.n_pixels
        try:  # phase 2: map the slots, store this rank's partial into its slot
            if rank != root:
                with cx.lock:
                    N.check(cx, cx.lib.nbx_ipc_open(cx.handle, handle[0], N.C.byref(base)))
                mapped = True
            torch.cuda.synchronize()
            plan.run(base.value + rank * npix * 8, mode=N.OUT_RAW_STORE_F64, on_device=True)  # synchronous
        except Exception as e:  # noqa: BLE001
            err = e
        if not _all_ok(err is None, group):  # every rank's stores are finished (or none started)
            raise err or RuntimeError("channel shard kernel failed on another rank")
        if rank == root:  # phase 3: the root sums the slots in rank order
            try:
                result = out if out is not None else PixelBuffer.zeros(ctx.panel.dims, "f32")
                mode = N.OUT_F32 if result.precision == "f32" else N.OUT_F64
                bad = N.C.c_int64(-1)
                with cx.lock:
                    st = cx.lib.nbx_reduce_slots(cx.handle, base.value, world, npix, plan.scale, mode,
                                                 result.data.ctypes.data, 0, N.C.byref(bad))
                    N.check(cx, st, bad.value)
            except Exception as e:  # noqa: BLE001
                err = e
        if not _all_ok(err is None, group):  # the root has read every slot
            raise err or RuntimeError("channel shard reduction failed on the root")
    finally:
        if plan is not None:
            plan.close()
        if mapped:
            with cx.lock:
                if rank == root:
                    cx.lib.nbx_ipc_free(cx.handle, base)
                else:
                    cx.lib.nbx_ipc_close(cx.handle, base)
    return result


def _native_channel_sharded(ctx: SpotsContext, out: PixelBuffer | None, group, root: int, rank: int):
    """The whole exchange inside the C ABI: nbx_spots_reduce with torch's NCCL communicator
    (every rank its shard's partial, ncclReduce to the root, scale + store on the root)."""
    import torch
    import torch.distributed as dist

    from .kernels import describe

    pg = group if group is not None else dist.distributed_c10d._get_default_group()
    backend = pg._get_backend(torch.device("cuda"))
    if not hasattr(backend, "_comm_ptr"):
        raise ValueError("transport='native' needs an NCCL process group")
    flag = torch.zeros(1, device="cuda")
    dist.all_reduce(flag, group=group)  # NCCL groups create their communicator on first use
    torch.cuda.synchronize()
    comm = backend._comm_ptr()
    dev = torch.cuda.current_device()
    cx = N.context(dev)
    desc = describe(ctx)
    result = None
    addr, mode = None, N.OUT_F32
    if rank == root:
        result = out if out is not None else PixelBuffer.zeros(ctx.panel.dims, "f32")
        addr, mode = result.data.ctypes.data, (N.OUT_F32 if result.precision == "f32" else N.OUT_F64)
    bad = N.C.c_int64(-1)
    with cx.lock:
        st = cx.lib.nbx_spots_reduce(cx.handle, N.C.byref(desc.c), N.COMPUTE[getattr(ctx, "compute", "fp64")],
                                     N.C.c_void_p(comm), root, mode, addr, 0, N.C.byref(bad))
        N.check(cx, st, bad.value)
    return result


def simulate_channel_sharded(ctx: SpotsContext, out: PixelBuffer | None = None, *, group=None, root: int = 0,
                             partial: Callable | None = None, finalize: Callable | None = None,
                             transport: str = "nccl"):
    """One image split by energy channel over the ranks of ``group``; returns the image on root, else None.

    ``root`` is a rank WITHIN ``group`` (translated to the global rank for the collectives).
    ``transport="nccl"`` (default, the north star's NCCL reduce): partial images in CUDA
    tensors, one ``dist.reduce`` to the root, scale + store there.  ``transport="p2p"``: the
    partials are stored by each rank's kernel directly into the root's memory (CUDA IPC /
    NVLink peer stores) and summed there in rank order -- no separate collective.
    ``transport="native"``: the same NCCL reduce issued by the C ABI (nbx_spots_reduce) on
    torch's NCCL communicator -- what a C caller of the library does with its own ncclComm_t.
    ``partial(ctx, lo, hi, norm) -> (raw_tensor, scale)`` and ``finalize(raw_tensor, scale,
    out)`` (NCCL transport) default to the GPU library.
    """
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    if not 0 <= root < world:
        raise ValueError(f"root {root} is not a rank of the group (size {world})")
    if transport not in ("nccl", "p2p", "native"):
        raise ValueError("transport must be 'nccl', 'p2p' or 'native'")
    n_src = len(ctx.spectrum.samples)
    if n_src < world:
        raise ValueError(f"{n_src} sources cannot be split over {world} ranks")
    if transport == "p2p" and world > 1:
        return _p2p_channel_sharded(ctx, out, group, root, world, rank)
    if transport == "native":
        return _native_channel_sharded(ctx, out, group, root, rank)
    if world == 1 and partial is None and finalize is None:
        # one shard is the whole spectrum: the single-image call (same arithmetic -- unscaled
        # FP64 sum, one scale, one cast -- with the row-banded download overlapping the kernel)
        from .kernels import nanobragg_spots

        if out is None:
            out = PixelBuffer.zeros(ctx.panel.dims, "f32")
        nanobragg_spots(ctx, out)
        return out
    partial = partial or _gpu_partial
    finalize = finalize or _gpu_finalize
    lo, hi = channel_shards(n_src, world)[rank]
    raw, scale = partial(ctx, lo, hi, global_norm(ctx))
    if world > 1:
        dist.reduce(raw, dst=_global_rank(group, root), op=dist.ReduceOp.SUM, group=group)
    if rank != root:
        return None
    if out is None:
        out = PixelBuffer.zeros(ctx.panel.dims, "f32")
    finalize(raw, scale, out)
    return out
