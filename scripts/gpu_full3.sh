timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
tail -2 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench exit $?"
python -c "
import json; d=json.load(open('gpurun_out/bench.json')); print(d['value'], d['stages'], d['h_matvec']['s1']['GB/s']); print({k: v['ms'] for k, v in d['kernel_ledger'].items()})"
timeout 900 python scripts/bench_configs.py 3 > gpurun_out/configs.log 2>&1; echo "configs exit $?"
python -c "
import json
for l in open('gpurun_out/configs.log'):
    if l.startswith('{'): d=json.loads(l); print(d['config'], round(d['s_per_iteration'],4), d['stages_s'])"
