"""bench.py's multi-rank control flow on a one-GPU box.

Two torchrun ranks share cuda:0 with gloo collectives (NBX_BENCH_SHARE_GPU=1, test-only):
image sharding (independent images per rank, barrier + max-over-ranks timing, e2e on every
rank) and channel sharding (FP64 partials reduced to rank 0, finalize) each print one
well-formed JSON line for the whole job.  Real runs put one rank per GPU over NCCL.
"""
import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def torchrun(args, port):
    env = dict(os.environ, NBX_BENCH_SHARE_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(ROOT / "bench.py"), "--gpus", "2", *args]
    res = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert res.returncode == 0, res.stderr[-3000:]
    lines = [ln for ln in res.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, res.stdout  # rank 0 alone prints
    return json.loads(lines[0])


def test_image_sharded_two_ranks(gpu):
    d = torchrun(["--steps", "2", "--warmup", "3", "--size", "512", "--no-extras"], 29531)
    assert d["n_gpus"] == 2 and d["scaling"] == "weak" and d["config"]["global_batch"] == 2
    assert d["value"] > 0 and d["gpu_launches"] == 2 * 2  # whole job: 2 steps x 2 ranks


@pytest.mark.parametrize("transport", ["nccl", "p2p"])
def test_channel_sharded_two_ranks(gpu, transport):
    d = torchrun(["--mode", "channels", "--channels", "64", "--steps", "2", "--warmup", "3", "--size", "512",
                  "--transport", transport], 29532 if transport == "nccl" else 29536)
    assert d["n_gpus"] == 2 and d["scaling"] == "strong" and d["config"]["images_per_gpu_per_step"] == 0.5
    assert d["value"] > 0 and d["e2e"]["value"] > 0
    assert d["gpu_launches"] == 2 * 2 + 2  # 2 steps x 2 ranks + one root reduction per step


CAMPAIGN_SCRIPT = r'''
import os, sys, json
sys.path.insert(0, os.environ["NBX_ROOT"])
import torch.distributed as dist
from paper_2205_07976_b200 import synthetic
from paper_2205_07976_b200.io import run_campaign, read_image
dist.init_process_group("gloo")
panel = synthetic.roi(synthetic.rayonix_panel(), 1800, 1800, 48, 64)
ctx_for = lambda i: synthetic.ls49_context(synthetic.SEED + i, panel=panel, n_channels=4, n_domains=2)
res = run_campaign(ctx_for, 7, sys.argv[1], first_image=3)
print(json.dumps({"rank": dist.get_rank(), "indices": res.indices, "crcs": res.crcs}), flush=True)
dist.destroy_process_group()
'''


def test_campaign_sharded_over_two_ranks(gpu, tmp_path):
    """run_campaign under torchrun: each rank renders a contiguous share of
    the 7 images (plan_batches: 4 + 3), the shares cover every index once, and every image
    equals a one-rank campaign's bit for bit (same CRC)."""
    script = tmp_path / "camp.py"
    script.write_text(CAMPAIGN_SCRIPT)
    env = dict(os.environ, NBX_ROOT=str(ROOT))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", "29533", str(script), str(tmp_path / "two")]
    res = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stderr[-3000:]
    rows = sorted((json.loads(ln) for ln in res.stdout.splitlines() if ln.startswith("{")), key=lambda r: r["rank"])
    assert [r["indices"] for r in rows] == [[3, 4, 5, 6], [7, 8, 9]]
    crc2 = {i: c for r in rows for i, c in zip(r["indices"], r["crcs"])}
    one = subprocess.run([sys.executable, str(script), str(tmp_path / "one")], capture_output=True, text=True,
                         timeout=600, env=dict(env, RANK="0", WORLD_SIZE="1", MASTER_ADDR="127.0.0.1",
                                               MASTER_PORT="29534"))
    assert one.returncode == 0, one.stderr[-3000:]
    r1 = json.loads([ln for ln in one.stdout.splitlines() if ln.startswith("{")][0])
    assert dict(zip(r1["indices"], r1["crcs"])) == crc2


P2P_SCRIPT = r'''
import os, sys, json
sys.path.insert(0, os.environ["NBX_ROOT"])
import numpy as np
import torch, torch.distributed as dist
from paper_2205_07976_b200 import PixelBuffer, nanobragg_spots, parallel, synthetic
dist.init_process_group("gloo")
torch.cuda.set_device(0)
panel = synthetic.roi(synthetic.rayonix_panel(), 1880, 1880, 40, 48)
res = {}
for compute in ("fp64", "fp32"):
    ctx = synthetic.ls49_context(panel=panel, n_channels=9, n_domains=3, compute=compute)
    a = parallel.simulate_channel_sharded(ctx, PixelBuffer.zeros(panel.dims, "f64"), transport="p2p")
    b = parallel.simulate_channel_sharded(ctx, PixelBuffer.zeros(panel.dims, "f64"), transport="nccl")
    if dist.get_rank() == 0:
        whole = PixelBuffer.zeros(panel.dims, "f64")
        nanobragg_spots(ctx, whole)
        res[compute] = {"p2p_vs_reduce": float(np.abs(a.data - b.data).max() / np.abs(b.data).max()),
                        "p2p_vs_whole": float(np.abs(a.data - whole.data).max() / np.abs(whole.data).max())}
    else:
        assert a is None and b is None
if dist.get_rank() == 0:
    print(json.dumps(res), flush=True)
dist.destroy_process_group()
'''


def test_p2p_channel_sharded_transport_two_ranks(gpu, tmp_path):
    """The fused peer-memory transport for channel shards (each rank's kernel stores its partial
    into the root's IPC-mapped slot; the root sums slots in rank order) equals the reduce-based
    path and the whole image (both ranks on one GPU here; NVLink peers on a real box)."""
    script = tmp_path / "p2p.py"
    script.write_text(P2P_SCRIPT)
    env = dict(os.environ, NBX_ROOT=str(ROOT))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", "29535", str(script)]
    res = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stderr[-3000:]
    d = json.loads([ln for ln in res.stdout.splitlines() if ln.startswith("{")][0])
    assert d["fp64"]["p2p_vs_reduce"] < 1e-15 and d["fp64"]["p2p_vs_whole"] < 1e-12, d
    assert d["fp32"]["p2p_vs_reduce"] < 1e-15 and d["fp32"]["p2p_vs_whole"] < 1e-4, d


P2P_FAIL_SCRIPT = r'''
import os, sys, json
sys.path.insert(0, os.environ["NBX_ROOT"])
import numpy as np
import torch, torch.distributed as dist
from paper_2205_07976_b200 import PixelBuffer, nanobragg_spots, parallel, synthetic
from paper_2205_07976_b200 import kernels as K
dist.init_process_group("gloo")
torch.cuda.set_device(0)
rank = dist.get_rank()
panel = synthetic.roi(synthetic.rayonix_panel(), 1880, 1880, 24, 32)
ctx = synthetic.ls49_context(panel=panel, n_channels=6, n_domains=2, compute="fp64")
out = {}
orig_run = K.SpotsPlan.run
for phase, failing in (("kernel", 1), ("kernel", 0), ("setup", 1)):
    def boom(self, *a, **k):
        raise RuntimeError("injected kernel failure")
    orig_init = K.SpotsPlan.__init__
    def bad_init(self, *a, **k):
        raise RuntimeError("injected set-up failure")
    if rank == failing:
        if phase == "kernel":
            K.SpotsPlan.run = boom
        else:
            K.SpotsPlan.__init__ = bad_init
    try:
        parallel.simulate_channel_sharded(ctx, PixelBuffer.zeros(panel.dims, "f64"), transport="p2p")
        out[f"{phase}{failing}"] = "no error"
    except RuntimeError as e:
        out[f"{phase}{failing}"] = str(e)
    K.SpotsPlan.run = orig_run
    K.SpotsPlan.__init__ = orig_init
# after the failures the transport still works (slots freed, nothing left mapped)
a = parallel.simulate_channel_sharded(ctx, PixelBuffer.zeros(panel.dims, "f64"), transport="p2p")
if rank == 0:
    whole = PixelBuffer.zeros(panel.dims, "f64")
    nanobragg_spots(ctx, whole)
    out["after"] = float(np.abs(a.data - whole.data).max() / np.abs(whole.data).max())
print(json.dumps({"rank": rank, **out}), flush=True)
dist.destroy_process_group()
'''


def test_p2p_channel_sharded_failure_on_one_rank(gpu, tmp_path):
    """a rank failing in set-up or in its kernel makes EVERY rank raise (the failing
    one its own error, the others 'failed on another rank') instead of hanging in a barrier or
    freeing slots a peer still writes; the transport works again afterwards."""
    script = tmp_path / "p2p_fail.py"
    script.write_text(P2P_FAIL_SCRIPT)
    env = dict(os.environ, NBX_ROOT=str(ROOT))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", "29537", str(script)]
    res = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=300)
    assert res.returncode == 0, res.stderr[-3000:]
    rows = {r["rank"]: r for r in (json.loads(ln) for ln in res.stdout.splitlines() if ln.startswith("{"))}
    for key, failing in (("kernel1", 1), ("kernel0", 0), ("setup1", 1)):
        for rank in (0, 1):
            msg = rows[rank][key]
            if rank == failing:
                assert msg.startswith("injected"), (key, rank, msg)
            else:
                assert "another rank" in msg, (key, rank, msg)
    assert rows[0]["after"] < 1e-12


NATIVE_SCRIPT = r'''
import ctypes as C, os, sys, json
sys.path.insert(0, os.environ["NBX_ROOT"])
import numpy as np
import torch, torch.distributed as dist
from paper_2205_07976_b200 import PixelBuffer, describe, nanobragg_spots, parallel, synthetic
from paper_2205_07976_b200 import _native as N
torch.cuda.set_device(0)
dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
panel = synthetic.roi(synthetic.rayonix_panel(), 1880, 1880, 40, 48)
res = {}
for compute in ("fp64", "fp32"):
    ctx = synthetic.ls49_context(panel=panel, n_channels=9, n_domains=3, compute=compute)
    got = parallel.simulate_channel_sharded(ctx, PixelBuffer.zeros(panel.dims, "f32"), transport="native")
    whole = PixelBuffer.zeros(panel.dims, "f32")
    nanobragg_spots(ctx, whole)
    res[compute] = {"bitwise": bool(np.array_equal(got.data, whole.data)),
                    "rel": float(np.abs(got.data.astype(float) - whole.data).max() / whole.data.max())}
# the C ABI's argument checks
cx = N.context(0)
desc = describe(synthetic.ls49_context(panel=panel, n_channels=9, n_domains=3, compute="fp64"))
bad = C.c_int64(-1)
out = np.zeros(panel.n_pixels, np.float32)
comm = dist.distributed_c10d._get_default_group()._get_backend(torch.device("cuda"))._comm_ptr()
res["null_comm"] = cx.lib.nbx_spots_reduce(cx.handle, C.byref(desc.c), 0, None, 0, N.OUT_F32, out.ctypes.data, 0,
                                           C.byref(bad))
res["bad_root"] = cx.lib.nbx_spots_reduce(cx.handle, C.byref(desc.c), 0, C.c_void_p(comm), 1, N.OUT_F32,
                                          out.ctypes.data, 0, C.byref(bad))
print(json.dumps(res), flush=True)
dist.destroy_process_group()
'''


def test_native_nccl_reduce_single_rank(gpu, tmp_path):
    """nbx_spots_reduce (the C ABI's channel-sharded image over a caller's ncclComm_t) with torch's
    one-rank NCCL communicator: the image equals nanobragg_spots bit for bit on both paths (one
    shard = the whole spectrum, the same global scale); a NULL communicator or a root outside the
    communicator is an argument error.  (NCCL refuses two ranks on one GPU: the multi-rank
    arithmetic -- shards, global norm, reduce, root-side scale -- is the gloo world-8 suite's.)"""
    script = tmp_path / "native.py"
    script.write_text(NATIVE_SCRIPT)
    env = dict(os.environ, NBX_ROOT=str(ROOT))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1", "--master-addr",
           "127.0.0.1", "--master-port", "29538", str(script)]
    res = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=300)
    assert res.returncode == 0, res.stderr[-3000:]
    d = json.loads([ln for ln in res.stdout.splitlines() if ln.startswith("{")][0])
    assert d["fp64"]["bitwise"] and d["fp32"]["rel"] < 1e-6, d
    assert d["null_comm"] == 1 and d["bad_root"] == 1, d
