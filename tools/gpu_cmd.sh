mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_xtrace.py tests/test_gpu_spots.py -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "rc=$?" >> gpurun_out/bench.err
tail -3 gpurun_out/pytest_gpu.log; python -c "
import json; d=json.load(open('gpurun_out/bench.json')); print(d['value'], d['e2e']['value'], d.get('e2e_reference_objects'))"; tail -3 gpurun_out/bench.err
