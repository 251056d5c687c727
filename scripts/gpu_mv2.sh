timeout 900 python -m pytest tests/test_gpu_hmatvec.py tests/test_gpu_hodlr.py -x -q > gpurun_out/pytest_mv.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_mv.log
tail -2 gpurun_out/pytest_mv.log
timeout 600 python scripts/probe_matvec.py 4 2 1 > gpurun_out/probe_mv.log 2>&1; cat gpurun_out/probe_mv.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench exit $?"
python -c "
import json; d=json.load(open('gpurun_out/bench.json')); print(d['value'], d['e2e']['value'], d['stages'], d['h_matvec'], d['gpu_launches'])"
