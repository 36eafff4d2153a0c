"""Summarise an ncu --set full report: time, DRAM bytes, pipe utilisation, issue, top stall reasons.

usage: python tools/ncu_summary.py gpurun_out/prof_fp32.ncu-rep [--json]
"""
import csv
import json
import re
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, units, vals = rows[0], rows[1], rows[2]
get = {h: (v, u) for h, u, v in zip(hdr, units, vals)}


def num(name):
    v, u = get.get(name, ("nan", ""))
    try:
        x = float(v.replace(",", ""))
    except ValueError:
        return float("nan")
    scale = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1, "ms": 1e-3, "us": 1e-6, "ns": 1e-9,
             "usecond": 1e-6, "msecond": 1e-3, "nsecond": 1e-9}.get(u, 1)
    return x * scale


out = {
    "kernel": get.get("Kernel Name", ("?", ""))[0],
    "duration_s": num("gpu__time_duration.sum"),
    "dram_bytes_read": num("dram__bytes_read.sum"),
    "dram_bytes_write": num("dram__bytes_write.sum"),
    "registers": num("launch__registers_per_thread"),
    "warps_active_pct": num("sm__warps_active.avg.pct_of_peak_sustained_active"),
    "issue_active_pct": num("smsp__issue_active.avg.pct_of_peak_sustained_active"),
    "inst_executed": num("smsp__inst_executed.sum"),
    "sm_clock_hz": num("sm__cycles_elapsed.avg.per_second"),
}
out["dram_bytes_per_launch"] = out["dram_bytes_read"] + out["dram_bytes_write"]
# executed FP-pipe thread operations of the launch (predicated-on lanes only; an FMA counts once):
# the measured work behind bench.py's roofline.achieved, and its fraction of the pipe's lane peak
cyc = num("smsp__cycles_elapsed.avg")
for prec, ops in (("fp64", ("dadd", "dfma", "dmul")), ("fp32", ("fadd", "ffma", "fmul"))):
    rate = sum(num(f"smsp__sass_thread_inst_executed_op_{o}_pred_on.sum.per_cycle_elapsed") for o in ops)
    if rate == rate and cyc == cyc:
        out[f"{prec}_thread_ops"] = rate * cyc
        out[f"{prec}_thread_ops_per_cycle"] = round(rate, 2)
peak64 = num("sm__sass_thread_inst_executed_op_dfma_pred_on.sum.peak_sustained")
if peak64 == peak64 and "fp64_thread_ops_per_cycle" in out:
    out["fp64_peak_ops_per_cycle"] = peak64
    out["fp64_ops_frac_of_peak"] = round(out["fp64_thread_ops_per_cycle"] / peak64, 4)
pipes = {}
for h in hdr:
    m = re.match(r"sm__inst_executed_pipe_(\w+)\.avg\.pct_of_peak_sustained_active$", h)
    if m and num(h) > 0.5:
        pipes[m.group(1)] = round(num(h), 2)
    m = re.match(r"sm__pipe_(\w+)_cycles_active\.avg\.pct_of_peak_sustained_active$", h)
    if m and num(h) > 0.5:
        pipes["cycles_" + m.group(1)] = round(num(h), 2)
out["pipes_pct"] = pipes
stalls = {}
for h in hdr:
    m = re.match(r"smsp__pcsamp_warps_issue_stalled_(\w+)$", h)
    if m and not m.group(1).endswith("not_issued"):
        stalls[m.group(1)] = num(h)
tot = sum(v for v in stalls.values() if v == v) or 1
out["stall_share"] = {k: round(v / tot, 3) for k, v in sorted(stalls.items(), key=lambda kv: -kv[1])[:8]}
if "--json" in sys.argv:
    print(json.dumps(out))
else:
    for k, v in out.items():
        print(f"{k:24s} {v}")
