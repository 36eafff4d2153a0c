"""Digest an ncu --set full capture of a spot kernel into profiles/ and point profiles/ncu_summary.json
(the record bench.py's roofline reads) at it.

usage: python tools/update_ncu_summary.py <report.ncu-rep> <fp64|fp32> <profile-name> <kernel_variant> <steps>
  e.g. python tools/update_ncu_summary.py gpurun_out/prof_fp64.ncu-rep fp64 r02_v2_spots_fp64_ncu 6 73728000000
The capture must be of the C2 workload (tools/quick_perf.py 3840 <compute>): bench.py uses its
FP64 op count only when kernel_variant and steps match its own plan.
"""
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
rep, compute, name, variant, steps = sys.argv[1:6]
digest = json.loads(subprocess.run([sys.executable, str(ROOT / "tools" / "ncu_summary.py"), rep, "--json"],
                                   capture_output=True, text=True, check=True).stdout)
digest["kernel_variant"] = int(variant)
digest["steps_per_launch"] = int(float(steps))
if "fp64_thread_ops" in digest:
    digest["fp64_ops_per_step"] = digest["fp64_thread_ops"] / digest["steps_per_launch"]
out = ROOT / "profiles" / f"{name}.json"
out.write_text(json.dumps(digest, indent=1) + "\n")
summ_path = ROOT / "profiles" / "ncu_summary.json"
summ = json.loads(summ_path.read_text()) if summ_path.exists() else {}
keep = ("dram_bytes_per_launch", "pipes_pct", "duration_s", "kernel", "kernel_variant", "steps_per_launch",
        "fp64_thread_ops", "fp64_ops_per_step", "fp64_ops_frac_of_peak", "issue_active_pct", "inst_executed")
summ[f"spots_{compute}"] = {k: digest[k] for k in keep if k in digest} | {"source": f"profiles/{name}.json"}
summ_path.write_text(json.dumps(summ, indent=1) + "\n")
print(json.dumps(summ[f"spots_{compute}"], indent=1))
