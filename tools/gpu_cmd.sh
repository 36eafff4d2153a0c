mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python tools/fp32_variants.py > gpurun_out/fp32v.log 2>&1
tail -5 gpurun_out/pytest_gpu.log; cat gpurun_out/fp32v.log
