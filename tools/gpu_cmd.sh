mkdir -p gpurun_out
rm -f gpurun_out/rec_error.log
for v in default mb5; do
  if [ $v = default ]; then unset NBX_LIB; else export NBX_LIB=$PWD/variants/$v/libnbx.so; fi
  echo "== $v" >> gpurun_out/rec_error.log
  timeout 300 python tools/rec_error.py --full >> gpurun_out/rec_error.log 2>&1
done
unset NBX_LIB
timeout 900 python -m pytest tests/test_gpu_segmented.py tests/test_gpu_spots.py tests/test_gpu_fullsize.py tests/test_gpu_fuzz.py -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
grep -v "bracket\|^seed [12]" gpurun_out/rec_error.log; tail -4 gpurun_out/pytest_gpu.log
