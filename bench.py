"""Benchmark: LS49-shape spot images (BASELINE.json configs[1], C2) on 1..8 B200s.

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]
    torchrun --nproc-per-node N bench.py --gpus N ...   (one rank per GPU, image-sharded)

One step = one full C2 image per GPU (3840 x 3840 pixels, 100 energy channels,
50 mosaic domains, oversample 1: 7.3728e10 pixel x source x mosaic steps),
each image with its own orientation / mosaic / weight seed (C3 sharding: no
collective).  `value` is whole-job images/s with every input resident in HBM
(device time, CUDA events, max over ranks); `e2e` is the same metric through
the drop-in nanobragg_spots() call with host buffers (descriptor upload and
image download inside the timed region).  Prints ONE JSON line on rank 0.

--impl reference times the reference's own CPU implementation (xtrace from
baseline/_ref, NumPy FP64, one forked process per host core on row stripes,
SURVEY §8 D1) on a bounded sample of the same workload; the C oracle port is
used if baseline/_ref is absent.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "images/s and Gsteps/s (pixel×source×mosaic×subpixel) at 1/2/4/8 B200"
WORKLOAD = "C2 LS49-shape image: 3840x3840 Rayonix-like, 100 energy channels, 50 mosaic domains, oversample 1"
STEP_INSTR = 126  # FP-pipe instructions per step, SURVEY §8 D1 (FMA = 1)
# What the implementation actually issues per step on its bounding pipe, counted in the
# SASS of the hot loop (tools/sass_loop.py), by nbx_plan_info_t.kernel_variant:
#   (pipe, pipe lane-ops per step, lanes per SM per clock of that pipe)
IMPL_OPS = {1: ("fma", 41, 128), 5: ("fma", 59, 128), 2: ("fma", 65, 128), 0: ("fp64", 73, 64), 4: ("fp64", 22, 64),
            6: ("fp64", 18, 64)}  # 6: 21 with Reinsch numerators, 18 with Chebyshev ones (76% of C2's warp-runs)
SMS = 148


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    # fp64 = the reference's own arithmetic (kernels.py:247-273 computes in float64) and the drop-in's
    # default for a reference SpotsContext: the headline.  fp32 is reported beside it (fp32_path).
    ap.add_argument("--compute", default="fp64", choices=["fp32", "fp64"])
    ap.add_argument("--size", type=int, default=3840)
    ap.add_argument("--channels", type=int, default=100)
    ap.add_argument("--domains", type=int, default=50)
    ap.add_argument("--mode", default="image", choices=["image", "channels", "jungfrau"],
                    help="image: C2 image-sharded (default); channels: C5 one 1000-channel image channel-sharded; "
                         "jungfrau: C4 256-panel FP64")
    ap.add_argument("--no-extras", action="store_true", help="skip e2e / fp64 / cpu-baseline legs")
    ap.add_argument("--transport", default="nccl", choices=["nccl", "p2p"],
                    help="channels mode: NCCL reduce of the partials (default) or fused peer-memory slots")
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 50 ms; only samples received between
    mark_start() and mark_end() (the timed region) are summarised.  The sampler is started and
    has produced its first line before the timed region begins."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines: list[tuple[float, str]] = []
        self.window = (None, None)

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-i",
                 str(self.device), "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            t_end = time.monotonic() + 3.0
            while not self.lines and time.monotonic() < t_end and self.proc.poll() is None:
                time.sleep(0.01)
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.monotonic(), line.strip()))

    def mark_start(self):
        self.window = (time.monotonic(), None)

    def mark_end(self):
        self.window = (self.window[0], time.monotonic())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        mhz, maxes, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        t0, t1 = self.window
        inside = [ln for t, ln in self.lines if (t0 is None or t >= t0) and (t1 is None or t <= t1)]
        for ln in inside or [ln for _, ln in self.lines]:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                mhz.append(float(parts[0]))
                maxes.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        load = [m for m in mhz if m > 300] or mhz
        return {"sm_mhz": statistics.median(load) if load else None,
                "sm_max_mhz": max(maxes) if maxes else None,
                "reasons": sorted(reasons), "samples": len(mhz)}


# ----------------------------------------------------------------------------- our arm
def run_ours(args):
    if args.mode == "channels" and args.channels == 100:
        args.channels = 1000
    if args.mode == "jungfrau" and args.compute == "fp32" and "--compute" not in sys.argv:
        args.compute = "fp64"
    world, rank, local = dist_env()
    # NBX_BENCH_SHARE_GPU=1 (test only): every rank on cuda:0 with gloo collectives, to exercise
    # the multi-rank control flow on a one-GPU box; real runs are one rank per GPU over NCCL
    share = os.environ.get("NBX_BENCH_SHARE_GPU") == "1"
    if share:
        local = 0
    os.environ["NBX_DEVICE"] = str(local)
    import numpy as np
    import torch
    import torch.distributed as dist

    torch.cuda.set_device(local)
    if world > 1:
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    from oracle import oracle  # cpu_baseline leg only (the checker, never the thing measured)
    from paper_2205_07976_b200 import PixelBuffer, SpotsPlan, nanobragg_spots, synthetic
    from paper_2205_07976_b200 import _native as N

    cx = N.context(local)
    # one non-default stream shared by torch (flush, events) and the library (kernels, copies)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    cx.lib.nbx_ctx_set_stream(cx.handle, N.C.c_void_p(stream.cuda_stream))

    from paper_2205_07976_b200 import parallel

    size = args.size
    r0 = (3840 - size) // 2
    panel = synthetic.rayonix_panel() if size == 3840 else synthetic.roi(synthetic.rayonix_panel(), r0, r0, size, size)
    mode = args.mode
    if mode == "jungfrau":
        panel = synthetic.jungfrau_detector()

    def ctx_for(i, compute):
        seed = synthetic.SEED + (0 if mode == "channels" else 100003 * rank) + i
        if mode == "jungfrau":
            return synthetic.jungfrau_context(seed, n_channels=args.channels, n_domains=args.domains,
                                              compute=compute)
        if mode == "channels":  # C5: 1000 channels, E_j = 7020 + 0.2 j eV
            return synthetic.ls49_context(seed, n_channels=args.channels, n_domains=args.domains, e0=7020.0,
                                          de=0.2, panel=panel, compute=compute)
        return synthetic.ls49_context(seed, n_channels=args.channels, n_domains=args.domains, panel=panel,
                                      compute=compute)

    n_img = args.warmup + args.steps
    if mode == "channels":
        # every step renders ONE image with the whole job: this rank's channel shard
        lo, hi = parallel.channel_shards(args.channels, world)[rank]
        plans = []
        for i in range(n_img):
            c = ctx_for(i, args.compute)
            plans.append(SpotsPlan(c, device=local, src_begin=lo, src_end=hi, norm=parallel.global_norm(c)))
        raw = torch.zeros(plans[0].n_pixels, dtype=torch.float64, device="cuda")
        slots = None
        if args.transport == "p2p" and world > 1:  # root's IPC slots, mapped once by every rank
            slots = N.C.c_void_p()
            handle = [None]
            if rank == 0:
                hb = N.C.create_string_buffer(64)
                N.check(cx, cx.lib.nbx_ipc_alloc(cx.handle, world * plans[0].n_pixels * 8, N.C.byref(slots), hb))
                handle = [bytes(hb.raw)]
            dist.broadcast_object_list(handle, src=0)
            if rank != 0:
                N.check(cx, cx.lib.nbx_ipc_open(cx.handle, handle[0], N.C.byref(slots)))
    else:
        plans = [SpotsPlan(ctx_for(i, args.compute), device=local) for i in range(n_img)]
    steps_per_unit = plans[0].steps  # per rank per step
    out = torch.empty(plans[0].n_pixels, dtype=torch.float32, device="cuda")
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")  # > 126 MB L2

    def barrier():
        if world > 1:
            dist.barrier()

    def one_step(i):
        flush.zero_()
        if mode != "channels":
            plans[i].run(out.data_ptr(), mode=N.OUT_F32, on_device=True)
            return
        if slots is not None:  # fused: the kernel stores this rank's partial into the root's slot
            plans[i].run(slots.value + rank * plans[i].n_pixels * 8, mode=N.OUT_RAW_STORE_F64, on_device=True)
            dist.barrier()
            if rank == 0:
                bad = N.C.c_int64(-1)
                st = cx.lib.nbx_reduce_slots(cx.handle, slots.value, world, plans[i].n_pixels, plans[i].scale,
                                             N.OUT_F32, out.data_ptr(), 1, N.C.byref(bad))
                N.check(cx, st, bad.value)
            dist.barrier()
            return
        raw.zero_()
        plans[i].run(raw.data_ptr(), mode=N.OUT_RAW_F64, on_device=True)
        if world > 1:
            dist.reduce(raw, dst=0, op=dist.ReduceOp.SUM)
        if rank == 0:
            bad = N.C.c_int64(-1)
            st = cx.lib.nbx_finalize(cx.handle, raw.data_ptr(), raw.numel(), plans[i].scale, N.OUT_F32,
                                     out.data_ptr(), 1, N.C.byref(bad))
            N.check(cx, st, bad.value)

    for i in range(args.warmup):
        one_step(i)

    # roofline denominator: live FMA probe on this GPU (MEASURED_PEAKS.json has no FP32/FP64 figure)
    peak = N.C.c_double(0.0)
    cx.lib.nbx_probe_fma_peak(cx.handle, 1 if args.compute == "fp64" else 0, N.C.byref(peak))

    kernel_ms = []
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:  # sampler running before the ranks line up
        barrier()
        torch.cuda.synchronize()
        clocks.mark_start()
        ev0.record(stream)
        for i in range(args.warmup, n_img):
            one_step(i)
            kernel_ms.append(plans[i].kernel_ms)
        ev1.record(stream)
        torch.cuda.synchronize()
        clocks.mark_end()
    barrier()
    elapsed = ev0.elapsed_time(ev1)
    if world > 1:
        t = torch.tensor([elapsed], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed = float(t.item())
    total_images = args.steps if mode == "channels" else world * args.steps
    steps_per_image = steps_per_unit * (world if mode == "channels" else 1)
    value = total_images / (elapsed / 1e3)
    gsteps = total_images * steps_per_image / (elapsed / 1e3) / 1e9
    mean_kernel = statistics.fmean(kernel_ms)
    workload = {"image": WORKLOAD if size == 3840 else f"{WORKLOAD} (ROI {size}x{size})",
                "channels": f"C5 single LS49-shape image, {size}x{size}, {args.channels} channels (7020 + 0.2 j eV), "
                            f"{args.domains} mosaic domains, channel-sharded over {world} GPU(s) + "
                            f"{'peer-memory slots' if args.transport == 'p2p' else 'NCCL reduce'}",
                "jungfrau": f"C4 Jungfrau-16M-like: 256 panels x 254x254, oversample 2, 3 thickness layers, "
                            f"{args.channels} channels, {args.domains} domains"}[mode]
    parallelism = {"image": f"image-sharded x{world} (no collective)",
                   "jungfrau": f"image-sharded x{world} (no collective)",
                   "channels": (f"channel-sharded x{world}, FP64 partials stored by each rank's kernel into rank 0's "
                                f"peer-memory slots, summed on rank 0" if args.transport == "p2p" and world > 1 else
                                f"channel-sharded x{world}, FP64 partials reduced to rank 0 (NCCL), finalize on rank 0")}
    result = {
        "metric": METRIC, "value": value, "unit": "images/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": elapsed / args.steps, "higher_is_better": True,
        "scaling": "strong" if mode == "channels" else "weak",
        "vs_baseline": None, "dtype": "f32" if args.compute == "fp32" else "f64",
        "data": "synthetic (seeded LS49-shape crystal, Wilson Fhkl to 1.6 A, random orientation per image)",
        "config": {"workload": workload, "mode": mode,
                   "images_per_gpu_per_step": 1 if mode != "channels" else 1.0 / world,
                   "global_batch": world if mode != "channels" else 1, "steps_per_image": steps_per_image,
                   "compute": args.compute, "parallelism": parallelism[mode],
                   "l2": "256 MB buffer written between timed images (L2 flushed); Fhkl grid L2-resident by design"},
        "gsteps_per_s": gsteps,
        "kernel_ms_mean": mean_kernel,
        # whole job: one spot kernel per step on every rank (+ one finalize / slot reduction per
        # step on the root in channel mode); the L2 flush is torch's, not counted
        "gpu_launches": args.steps * world + (args.steps if mode == "channels" else 0),
        "clocks": clocks.summary(),
    }
    clk = result["clocks"].get("sm_mhz") or 1965.0
    result["roofline"] = roofline(plans[0], mean_kernel, peak.value, clk, args.compute, plans[0].n_pixels * 4)

    if not args.no_extras:
        # e2e: the public API with host buffers, descriptor upload and image download inside the timed region
        e2e_steps = max(1, min(args.steps, 3))
        ctxs = [ctx_for(1000 + i, args.compute) for i in range(e2e_steps + 1)]
        img = PixelBuffer.zeros(panel.dims, "f32")

        def e2e_call(c):
            if mode == "channels":
                parallel.simulate_channel_sharded(c, img, transport=args.transport)
            else:
                nanobragg_spots(c, img)

        e2e_call(ctxs[0])  # warm (host tables, context)
        barrier()
        torch.cuda.synchronize()
        ev0.record(stream)
        call_ms = []
        for c in ctxs[1:]:
            t_call = time.perf_counter()
            e2e_call(c)
            call_ms.append(round((time.perf_counter() - t_call) * 1e3, 2))
        ev1.record(stream)
        torch.cuda.synchronize()
        e2e_ms = ev0.elapsed_time(ev1) / e2e_steps
        if world > 1:  # every rank ran its own images (image mode) or its shard (channels): max over ranks
            t = torch.tensor([e2e_ms], device="cuda", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_ms = float(t.item())
        info = plans[0].info
        h2d = int(info.table_cells) * (4 if args.compute == "fp32" else 8) + args.channels * 16 + \
            args.domains * 72 + 160 * len(getattr(panel, "panels", (panel,)))
        result["e2e"] = {"value": 1e3 / e2e_ms * (1 if mode == "channels" else world), "unit": "images/s", "h2d_bytes_per_step": h2d,
                         "d2h_bytes_per_step": int(plans[0].n_pixels) * 4 + 8, "ms_per_step": e2e_ms,
                         "api": ("paper_2205_07976_b200.parallel.simulate_channel_sharded(ctx, PixelBuffer)"
                                 if mode == "channels" else
                                 "paper_2205_07976_b200.nanobragg_spots(ctx, PixelBuffer) -> nbx_spots C ABI"),
                         "note": "whole job: every rank simulates its own images, slowest rank's time" if
                         mode != "channels" and world > 1 else "whole job", "call_wall_ms": call_ms}

    if rank == 0 and not args.no_extras and mode == "image":
        # the other compute path on the same workload (FP32: the 1e-4 path; FP64: the 1e-9 path), kernel time,
        # roofline and its own e2e through nanobragg_spots with host buffers
        other = "fp32" if args.compute == "fp64" else "fp64"
        po = SpotsPlan(ctx_for(0, other), device=local)
        po.run(out.data_ptr(), mode=N.OUT_F32, on_device=True)
        mso = []
        for _ in range(3):
            flush.zero_()
            po.run(out.data_ptr(), mode=N.OUT_F32, on_device=True)
            mso.append(po.kernel_ms)
        peak_o = N.C.c_double(0.0)
        cx.lib.nbx_probe_fma_peak(cx.handle, 1 if other == "fp64" else 0, N.C.byref(peak_o))
        ko = statistics.fmean(mso)
        block = {"dtype": "f64" if other == "fp64" else "f32", "kernel_ms": ko, "images_per_s": 1e3 / ko,
                 "gsteps_per_s": po.steps / ko / 1e6,
                 "roofline": roofline(po, ko, peak_o.value, clk, other, po.n_pixels * 4)}
        po.close()
        octx = [ctx_for(2000 + i, other) for i in range(3)]
        img_o = PixelBuffer.zeros(panel.dims, "f32")
        nanobragg_spots(octx[0], img_o)
        torch.cuda.synchronize()
        ev0.record(stream)
        for c in octx[1:]:
            nanobragg_spots(c, img_o)
        ev1.record(stream)
        torch.cuda.synchronize()
        e2e_o = ev0.elapsed_time(ev1) / (len(octx) - 1)
        block["e2e"] = {"value": 1e3 / e2e_o, "unit": "images/s", "ms_per_step": e2e_o,
                        "api": "paper_2205_07976_b200.nanobragg_spots(ctx, PixelBuffer) -> nbx_spots C ABI"}
        result[f"{other}_path"] = block

    if rank == 0 and not args.no_extras and world == 1 and mode == "image" and args.compute == "fp64" \
            and _xtrace_available():
        # the same e2e with the REFERENCE's own objects (xtrace SpotsContext / PixelBuffer from
        # baseline/_ref) handed to the drop-in: what a reference caller patched per INTEGRATION.md gets
        import xtrace.kernels as xk
        import xtrace.model as xm

        xs = [to_xtrace(ctx_for(3000 + i, "fp64")) for i in range(3)]
        xtable = xs[0][0].sf_table  # one structure-factor table object for the campaign, as in the reference
        xs = [to_xtrace(ctx_for(3000 + i, "fp64"), xtable) for i in range(3)]
        xp = xm.DetectorPanel(panel.slow_pixels, panel.fast_pixels, panel.pixel_size, panel.distance,
                              tuple(panel.beam_center))
        xctx = [xk.SpotsContext(c, xp, b, oversample=1) for c, b in xs]
        xbuf = xk.PixelBuffer.zeros(xp.dims, "f32")
        nanobragg_spots(xctx[0], xbuf)
        torch.cuda.synchronize()
        ev0.record(stream)
        for c in xctx[1:]:
            nanobragg_spots(c, xbuf)
        ev1.record(stream)
        torch.cuda.synchronize()
        xms = ev0.elapsed_time(ev1) / (len(xctx) - 1)
        result["e2e_reference_objects"] = {
            "value": 1e3 / xms, "unit": "images/s", "ms_per_step": xms,
            "api": "paper_2205_07976_b200.nanobragg_spots(xtrace.kernels.SpotsContext, xtrace.kernels.PixelBuffer)",
            "note": "the reference's own input/output objects (baseline/_ref) through the drop-in, FP64"}

    if rank == 0 and not args.no_extras and world == 1 and mode == "image":
        result["stages"] = stage_timings(cx, N, torch, stream, ctx_for(0, args.compute), panel)

    if rank == 0 and not args.no_extras and world == 1:
        result["cpu_baseline"] = cpu_baseline_port(ctx_for(0, "fp64"), panel, steps_per_image, oracle)

    if rank == 0:
        print(json.dumps(result), flush=True)
    for p in plans:
        p.close()
    if world > 1:
        dist.destroy_process_group()


def roofline(plan, kernel_ms: float, peak_tflops: float, clk_mhz: float, compute: str, writeback_bytes: int) -> dict:
    """Roofline of the spot kernel on its bounding pipe.

    achieved = executed bounding-pipe lane-ops per step x steps / kernel time, as TFLOP/s with one pipe
    op = 2 FLOP (the FMA convention of the peak).  FP64: the ops per step are MEASURED -- ncu's
    predicated-on DADD+DFMA+DMUL thread instructions of the committed capture of the same kernel
    variant on the same workload (profiles/ncu_summary.json: every FP64 op of the launch, the per-run
    anchors and slow channels included) / its steps; without a matching capture, the SASS count of
    the channel loop (IMPL_OPS, an under-count).  FP32: the SASS count of the MUFU loop (41 FMA-pipe
    lane-ops per step; ncu's FP32 op counters do not see the packed f32x2 lanes).  peak = the live FMA
    probe of the same pipe on this GPU (MEASURED_PEAKS.json holds no FP32/FP64 figure); frac =
    achieved / peak.  d1_frac keeps SURVEY §8 D1's fixed 126 instructions per step (it exceeds 1:
    the implementation needs far fewer instructions per step than that nominal count).
    """
    variant = plan.info.kernel_variant
    pipe, ops, lanes = IMPL_OPS.get(variant, ("fp64" if compute == "fp64" else "fma", STEP_INSTR, 64))
    ops_basis = f"{ops} SASS-counted {pipe}-pipe ops per step in the channel loop (kernel variant {variant})"
    sps = plan.steps / (kernel_ms / 1e3)
    traffic = None
    prof = ROOT / "profiles" / "ncu_summary.json"
    ncu_pipe = None
    if prof.exists():
        try:
            rec = json.loads(prof.read_text()).get(f"spots_{compute}", {})
            traffic = rec.get("dram_bytes_per_launch")
            ncu_pipe = rec.get("pipes_pct", {}).get("cycles_fp64" if compute == "fp64" else "cycles_fma")
            if (pipe == "fp64" and rec.get("kernel_variant") == variant and rec.get("fp64_thread_ops")
                    and rec.get("steps_per_launch") == plan.steps):
                ops = rec["fp64_thread_ops"] / rec["steps_per_launch"]
                ops_basis = (f"{ops:.2f} fp64-pipe ops per step measured by ncu (DADD+DFMA+DMUL thread "
                             f"instructions of {rec.get('source')}, kernel variant {variant}, same workload)")
        except (ValueError, AttributeError):
            traffic = None
    achieved = 2.0 * ops * sps / 1e12
    d1 = 2.0 * STEP_INSTR * sps / 1e12
    return {
        "bound": "fp64_pipe" if pipe == "fp64" else "fp32_fma_pipe", "achieved": achieved, "peak": peak_tflops,
        "unit": "TFLOP/s", "frac": achieved / peak_tflops if peak_tflops else None, "traffic": traffic,
        "kernel_variant": variant, "pipe_ops_per_step": ops,
        "pipe_frac_nominal": sps * ops / (SMS * lanes * clk_mhz * 1e6),
        "ncu_pipe_active_pct": ncu_pipe,
        "d1_frac": d1 / peak_tflops if peak_tflops else None, "d1_instr_per_step": STEP_INSTR,
        "basis": f"{ops_basis} x steps / mean spot-kernel time (CUDA events), 1 op = 2 FLOP; peak = live {pipe} "
                 "FMA probe (nbx_probe_fma_peak) on this GPU; pipe_frac_nominal uses 148 SMs x lanes/SM x median "
                 "SM clock; ncu_pipe_active_pct = sm__pipe_" + ("fp64" if pipe == "fp64" else "fma") +
                 "_cycles_active of the committed capture (profiles/ncu_summary.json)",
        "traffic_note": "ncu dram read+write bytes of one spot launch (profiles/ncu_summary.json): the inputs are "
                        "read once (L2-resident); most of the image write-back is still in the 126 MB L2 when "
                        "the kernel ends, so traffic < write-back bytes",
        "writeback": {"bytes_per_image": int(writeback_bytes), "gbs": writeback_bytes / (kernel_ms / 1e3) / 1e9},
    }


def hbm_peak_gbs() -> tuple[float, str]:
    try:
        v = float(json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"])
        return v, "MEASURED_PEAKS.json hbm_gbs"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"


def stage_timings(cx, N, torch, stream, ctx, panel) -> dict:
    """Device time of the stages around the spot kernel on the same C2 detector:
    add_background, simulate_image's fused spots+background launch, add_array, image_stats /
    image_histogram, Poisson noise; HBM-bound ones against the HBM peak with their algorithmic bytes."""
    from paper_2205_07976_b200 import BackgroundProfile
    from paper_2205_07976_b200.kernels import _bg_descriptor, describe

    water = BackgroundProfile(points=((0.0, 2.57), (0.0365, 2.58), (0.07, 2.8), (0.12, 5.0), (0.162, 8.0),
                                      (0.2, 7.5), (0.25, 7.0), (0.3, 6.5), (0.35, 6.1), (0.4, 5.8), (0.45, 5.5),
                                      (0.5, 5.2)))
    n = panel.n_pixels
    f32 = torch.rand(n, dtype=torch.float32, device="cuda") * 100
    f64 = torch.zeros(n, dtype=torch.float64, device="cuda")
    out32 = torch.empty(n, dtype=torch.float32, device="cuda")
    bad = N.C.c_int64(-1)
    bg_desc = _bg_descriptor(water, panel, ctx.spectrum, 1.0)
    img_desc = describe(ctx, background=water, thickness_factor=1.0)
    four = (N.C.c_double * 4)()
    counts = (N.C.c_int64 * 64)()
    uo, oo = N.C.c_int64(0), N.C.c_int64(0)
    lib, h = cx.lib, cx.handle
    calls = {
        "add_background": (lambda: lib.nbx_background(h, N.C.byref(bg_desc.c), N.OUT_F32, out32.data_ptr(), 1,
                                                      N.C.byref(bad)), None),
        "simulate_image_fused": (lambda: lib.nbx_spots(h, N.C.byref(img_desc.c), N.COMPUTE[ctx.compute],
                                                       N.OUT_IMAGE_F64, f64.data_ptr(), 1, N.C.byref(bad)), None),
        "add_array": (lambda: lib.nbx_add_array(h, N.C.c_void_p(f64.data_ptr()), N.C.c_void_p(f32.data_ptr()),
                                                n, 1), 20 * n),
        "image_stats": (lambda: lib.nbx_image_stats(h, N.C.c_void_p(f32.data_ptr()), n, 0, 1, four), 4 * n),
        "image_histogram": (lambda: lib.nbx_image_histogram(h, N.C.c_void_p(f32.data_ptr()), n, 0, 1, 64, 0.0,
                                                            100.0, counts, N.C.byref(uo), N.C.byref(oo)), 4 * n),
        "poisson_noise": (lambda: lib.nbx_add_noise(h, N.C.c_void_p(f32.data_ptr()), N.C.c_void_p(out32.data_ptr()),
                                                    n, 0, 7, 0, 1), 8 * n),
    }
    peak, peak_src = hbm_peak_gbs()
    res = {"detector": f"C2 {panel.slow_pixels}x{panel.fast_pixels}", "hbm_peak_gbs": peak, "hbm_peak_source": peak_src}
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for name, (fn, nbytes) in calls.items():
        assert fn() == 0, name
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(3):
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 3
        row = {"ms": ms}
        if nbytes:
            row.update({"algorithmic_bytes": nbytes, "gbs": nbytes / ms / 1e6, "hbm_frac": nbytes / ms / 1e6 / peak})
        res[name] = row
    # F3: the pipelined campaign (fused spots+background per image, .bin + sidecar with CRC-32,
    # download/CRC/write of image i overlapped with image i+1's kernel), 4 images after one warm-up
    import shutil
    import tempfile

    from paper_2205_07976_b200.io import run_campaign
    from paper_2205_07976_b200 import synthetic

    out_dir = Path(tempfile.mkdtemp(prefix="nbx_bench_campaign_"))
    try:
        def cfor(i):
            return synthetic.ls49_context(synthetic.SEED + 5000 + i, panel=panel, compute=ctx.compute)

        run_campaign(cfor, 1, out_dir, background=water)
        r2 = run_campaign(cfor, 2, out_dir, first_image=1, background=water)
        r6 = run_campaign(cfor, 6, out_dir, first_image=1, background=water)
        steady = (r6.seconds - r2.seconds) / 4
        res["campaign"] = {"images": 6, "ms_per_image": 1e3 * r6.seconds / 6, "images_per_s": 6 / r6.seconds,
                           "steady_ms_per_image": 1e3 * steady,
                           "basis": "host wall time of io.run_campaign (nbx_campaign) incl. file writes; "
                                    "steady = (T(6 images) - T(2 images)) / 4: the per-image cost once the "
                                    "pipeline is full (fill + drain -- first plan, last download/CRC/write "
                                    "-- excluded)"}
    finally:
        shutil.rmtree(out_dir, ignore_errors=True)
    return res


def cpu_baseline_port(ctx, panel, steps_per_image, oracle):
    """The C oracle (FP64 scalar restatement) on all host cores over a bounded row sample of the image."""
    import dataclasses

    from paper_2205_07976_b200 import describe, synthetic

    per_pixel = steps_per_image // panel.n_pixels  # every pixel costs the same number of steps
    one = panel.panels[0] if hasattr(panel, "panels") and len(panel.panels) > 1 else panel
    # ~1.6e9 steps: about 10 s of CPU work on the box's 16 host cores, whatever the config
    rows = max(1, min(one.slow_pixels, round(1.6e9 / (one.fast_pixels * per_pixel))))
    r0 = one.slow_pixels // 2 - rows // 2
    sub = dataclasses.replace(ctx, panel=synthetic.roi(one, r0, 0, rows, one.fast_pixels))
    desc = describe(sub)
    cores = host_cores()
    t0 = time.perf_counter()
    oracle.spots(desc, "f32", nthreads=cores)
    dt = time.perf_counter() - t0
    sample_steps = rows * one.fast_pixels * per_pixel
    sps = sample_steps / dt
    return {"value": sps / steps_per_image, "unit": "images/s", "cores": cores, "kind": "port",
            "gsteps_per_s": sps / 1e9, "seconds": dt, "cpu": cpu_model(),
            "sample": f"rows {r0}-{r0 + rows - 1} x {one.fast_pixels} px (panel 0) x every sub-pixel/layer/source/"
                      f"domain ({sample_steps:.3g} steps) of the same image, oracle/nbx_oracle.c FP64, {cores} threads"}


# ----------------------------------------------------------------------------- reference arm
def _xtrace_available():
    ref = ROOT / "baseline" / "_ref"
    if (ref / "xtrace" / "kernels.py").exists():
        sys.path.insert(0, str(ref))
        return True
    return False


def run_reference(args):
    world, rank, local = dist_env()
    if rank != 0:
        return  # rank 0 alone runs the CPU reference; the others exit without work
    from paper_2205_07976_b200 import synthetic

    size = args.size
    panel = synthetic.rayonix_panel() if size == 3840 else synthetic.roi(
        synthetic.rayonix_panel(), (3840 - size) // 2, (3840 - size) // 2, size, size)
    ctx = synthetic.ls49_context(synthetic.SEED, n_channels=args.channels, n_domains=args.domains, panel=panel,
                                 compute="fp64")
    steps_per_image = panel.n_pixels * args.channels * args.domains
    cores = host_cores()
    rows_per_step = cores  # one full-width row per forked process per step
    kind = "reference" if _xtrace_available() else "port"
    step_fn = _reference_step_xtrace(ctx, panel, cores) if kind == "reference" else _reference_step_port(ctx, panel, cores)
    row0 = panel.slow_pixels // 2 - rows_per_step // 2
    for i in range(args.warmup):
        step_fn(row0 + i % 4, rows_per_step)
    times = []
    for i in range(args.steps):
        t0 = time.perf_counter()
        step_fn(row0, rows_per_step)
        times.append(time.perf_counter() - t0)
    sample_steps = rows_per_step * panel.fast_pixels * args.channels * args.domains
    sec = sum(times)
    sps = sample_steps * args.steps / sec
    value = sps / steps_per_image
    sample = (f"{rows_per_step} full-width rows ({rows_per_step}x{panel.fast_pixels} px) x {args.channels} sources x "
              f"{args.domains} domains = {sample_steps:.3g} steps per step")
    impl_desc = ("xtrace.kernels.nanobragg_spots (baseline/_ref, unmodified, NumPy FP64) in one forked process "
                 "per core on row-stripe sub-panels" if kind == "reference" else
                 "oracle/nbx_oracle.c FP64 restatement, one thread per core")
    line = {
        "metric": METRIC, "value": value, "unit": "images/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": sec / args.steps * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (same seeded LS49-shape workload)",
        "config": {"workload": WORKLOAD, "steps_per_image": steps_per_image, "impl": impl_desc},
        "impl": "reference", "gsteps_per_s": sps / 1e9,
        "cpu_baseline": {"value": value, "unit": "images/s", "cores": cores, "kind": kind, "sample": sample,
                         "cpu": cpu_model()},
        "e2e": {"value": value, "unit": "images/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def to_xtrace(ctx, xtable=None):
    """The reference's own objects (baseline/_ref/xtrace) for one of our SpotsContexts."""
    import numpy as np
    import xtrace.model as xm

    c = ctx.crystal
    if xtable is None:
        hkl, amp = c.sf_table.arrays()
        xtable = xm.StructureFactorTable({tuple(map(int, h)): float(a) for h, a in zip(hkl, amp)},
                                         default_f=c.sf_table.default_f)
    xcrystal = xm.CrystalModel(
        cell=xm.UnitCell(c.cell.a, c.cell.b, c.cell.c, c.cell.alpha, c.cell.beta, c.cell.gamma),
        orientation=xm.Orientation(c.orientation.u), n_cells=c.n_cells,
        mosaic=xm.MosaicDomainSet(np.array(c.mosaic.rotations)), sf_table=xtable)
    s = ctx.spectrum
    xbeam = xm.BeamSpectrum(samples=s.samples, fluence=s.fluence, polarization_on=s.polarization_on,
                            beam_direction=s.beam_direction)
    return xcrystal, xbeam


def _reference_step_xtrace(ctx, panel, cores):
    import multiprocessing as mp

    import xtrace.kernels as xk
    import xtrace.model as xm

    os.environ.setdefault("OMP_NUM_THREADS", "1")
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    xcrystal, xbeam = to_xtrace(ctx)
    fork = mp.get_context("fork")

    def one_row(r):
        p = xm.DetectorPanel(1, panel.fast_pixels, panel.pixel_size, panel.distance,
                             (panel.beam_center[0] - r, panel.beam_center[1]))
        xctx = xk.SpotsContext(xcrystal, p, xbeam, oversample=ctx.oversample)
        out = xk.PixelBuffer.zeros(p.dims)
        xk.nanobragg_spots(xctx, out)
        os._exit(0)

    def step(r0, rows):
        procs = [fork.Process(target=one_row, args=(r0 + i,)) for i in range(rows)]
        for p in procs:
            p.start()
        for p in procs:
            p.join()

    return step


def _reference_step_port(ctx, panel, cores):
    from oracle import oracle
    from paper_2205_07976_b200 import describe, synthetic

    import dataclasses

    def step(r0, rows):
        sub = dataclasses.replace(ctx, panel=synthetic.roi(panel, r0, 0, rows, panel.fast_pixels))
        oracle.spots(describe(sub), "f32", nthreads=cores)

    return step


if __name__ == "__main__":
    a = parse()
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)
