#!/bin/bash
# One consistent measurement snapshot of the current commit on one GPU -> gpurun_out/snap/.
# usage: bash tools/gpu_snapshot.sh <version, e.g. r02_v2> [quick]
# Order matters: the ncu captures of the spot kernels come first and are digested on the box into
# profiles/ (tools/update_ncu_summary.py), so the bench lines that follow read the op counts of
# the same build; the updated profiles/*.json are copied to gpurun_out/snap/profiles/.
V=${1:?version}
O=gpurun_out/snap
mkdir -p $O/profiles
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt 2>&1
for c in fp64 fp32; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:spots_kernel -s 1 -c 1 \
      -o $O/prof_$c -f python tools/quick_perf.py 3840 $c > $O/ncu_$c.log 2>&1; echo "rc=$?" >> $O/ncu_$c.log
done
timeout 300 python tools/update_ncu_summary.py $O/prof_fp64.ncu-rep fp64 ${V}_spots_fp64_ncu 6 73728000000 > $O/upd64.log 2>&1
timeout 300 python tools/update_ncu_summary.py $O/prof_fp32.ncu-rep fp32 ${V}_spots_fp32_ncu 1 73728000000 > $O/upd32.log 2>&1
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err; echo "rc=$?" >> $O/bench.err
timeout 600 python bench.py --mode jungfrau --steps 3 --warmup 3 > $O/bench_c4_jungfrau_fp64.json 2> $O/bench_c4.err
timeout 600 python bench.py --mode channels --steps 3 --warmup 3 > $O/bench_c5_channels.json 2> $O/bench_c5.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2> $O/bench_ref.err
timeout 600 python tools/parity_report.py > $O/parity.json 2> $O/parity.err
timeout 600 python tools/campaign_perf.py 10 > $O/campaign.json 2> $O/campaign.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-extras > $O/launches_bench.log 2>&1
if [ "$2" != quick ]; then
  for t in memcheck racecheck initcheck; do
    timeout 1200 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize_run.py > $O/$t.log 2>&1; echo "rc=$?" >> $O/$t.log
  done
fi
cp profiles/ncu_summary.json profiles/${V}_spots_fp64_ncu.json profiles/${V}_spots_fp32_ncu.json $O/profiles/ 2>/dev/null
for f in $O/*.json; do echo "== $f"; head -c 600 $f; echo; done
tail -n 3 $O/*.log
