mkdir -p gpurun_out
for v in default mb5 mb4; do
  if [ $v = default ]; then unset NBX_LIB; else export NBX_LIB=$PWD/variants/$v/libnbx.so; fi
  echo "== $v" >> gpurun_out/rec_error.log
  timeout 300 python tools/rec_error.py --full >> gpurun_out/rec_error.log 2>&1; echo "rc=$?" >> gpurun_out/rec_error.log
done
unset NBX_LIB
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
cat gpurun_out/rec_error.log; tail -5 gpurun_out/pytest_gpu.log
