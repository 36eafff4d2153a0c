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
    assert d["value"] > 0 and d["gpu_launches"] == 2


def test_channel_sharded_two_ranks(gpu):
    d = torchrun(["--mode", "channels", "--channels", "64", "--steps", "2", "--warmup", "3", "--size", "512"], 29532)
    assert d["n_gpus"] == 2 and d["scaling"] == "strong" and d["config"]["images_per_gpu_per_step"] == 0.5
    assert d["value"] > 0 and d["e2e"]["value"] > 0
