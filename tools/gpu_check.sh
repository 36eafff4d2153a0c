#!/bin/bash
# Run the GPU checks step by step with their own timeouts; logs land in gpurun_out/.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout ${PYTEST_TIMEOUT:-900} python -m pytest tests -m gpu -q ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for a in "$@"; do
  echo "== $a" >> gpurun_out/extra.log
  timeout 600 bash -c "$a" >> gpurun_out/extra.log 2>&1; echo "rc=$?" >> gpurun_out/extra.log
done
tail -3 gpurun_out/smoke.log; tail -30 gpurun_out/pytest_gpu.log; tail -40 gpurun_out/extra.log 2>/dev/null || true
