mkdir -p gpurun_out
rm -f gpurun_out/rec_error.log
for v in default u2 u3 u2mb5; do
  if [ $v = default ]; then unset NBX_LIB; else export NBX_LIB=$PWD/variants/$v/libnbx.so; fi
  echo "== $v" >> gpurun_out/rec_error.log
  timeout 300 python tools/rec_error.py --full-only >> gpurun_out/rec_error.log 2>&1; echo "rc=$?" >> gpurun_out/rec_error.log
done
unset NBX_LIB
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "rc=$?" >> gpurun_out/bench.err
cat gpurun_out/rec_error.log; python -c "
import json; d=json.load(open('gpurun_out/bench.json')); print({k:d[k] for k in ('value','ms_per_step','dtype')}, d['e2e']['value'], d['roofline']['frac'], d['fp32_path']['kernel_ms'], d['fp32_path']['e2e'])"
