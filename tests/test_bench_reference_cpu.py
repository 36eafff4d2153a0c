"""bench.py's reference arm (`--impl reference`) runs here on CPU, single process and under
torchrun with two ranks (rank 0 alone measures and prints), with the line the driver expects:
the same metric / unit / config workload as our arm, impl "reference", a cpu_baseline
describing the run and a zero-copy e2e object."""
import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
pytestmark = pytest.mark.skipif(not (ROOT / "baseline" / "_ref" / "xtrace").exists(),
                                reason="reference not installed in baseline/_ref")


def _lines(cmd):
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert res.returncode == 0, res.stderr[-3000:]
    return [json.loads(ln) for ln in res.stdout.splitlines() if ln.startswith("{")]


def _check(d, n_gpus):
    assert d["impl"] == "reference" and d["n_gpus"] == n_gpus and d["steps"] == 1 and d["warmup"] == 3
    assert d["unit"] == "images/s" and d["higher_is_better"] is True and d["value"] > 0
    assert d["config"]["workload"].startswith("C2 LS49-shape image")
    cb = d["cpu_baseline"]
    assert cb["kind"] in ("reference", "port") and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


def test_reference_arm_single_process():
    lines = _lines([sys.executable, "bench.py", "--impl", "reference", "--steps", "1", "--warmup", "3"])
    assert len(lines) == 1
    _check(lines[0], 1)


def test_reference_arm_under_torchrun_rank0_prints():
    lines = _lines([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                    "--master-addr", "127.0.0.1", "--master-port", "29562", "bench.py", "--impl", "reference",
                    "--gpus", "2", "--steps", "1", "--warmup", "3"])
    assert len(lines) == 1
    _check(lines[0], 2)
