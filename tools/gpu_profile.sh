#!/bin/bash
# Bench + ncu evidence on one GPU; everything lands in gpurun_out/.
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
if [ -z "$SKIP_NCU" ]; then
# launch list of the same command (cold-cache, serialised: compare shares, not absolutes)
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-extras > gpurun_out/launches_bench.log 2>&1; echo "launches rc=$?" >> gpurun_out/launches_bench.log
# one full capture per compute path of the spot kernel at the C2 size
for c in fp32 fp64; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:spots_kernel -s 1 -c 1 \
      -o gpurun_out/prof_$c -f python tools/quick_perf.py 3840 $c > gpurun_out/ncu_$c.log 2>&1; echo "ncu $c rc=$?" >> gpurun_out/ncu_$c.log
done
fi
cat gpurun_out/bench.json; tail -n 3 gpurun_out/bench.err; tail -n 2 gpurun_out/ncu_fp32.log; tail -n 2 gpurun_out/ncu_fp64.log
