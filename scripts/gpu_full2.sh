timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python scripts/probe_matvec.py 64 1 > gpurun_out/probe_mv.log 2>&1; cat gpurun_out/probe_mv.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench exit $?"
python -c "
import json; d=json.load(open('gpurun_out/bench.json')); print(d['value'], d['e2e']['value'], d['stages'], d['h_matvec']['s1']['GB/s'], d['gpu_launches']); print(d['kernel_ledger'])"
timeout 900 python scripts/prof_detail.py 20 > gpurun_out/prof_detail.log 2>&1; echo "detail exit $?"
