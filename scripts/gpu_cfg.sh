timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
tail -2 gpurun_out/pytest_gpu.log
timeout 900 python scripts/bench_configs.py 3 > gpurun_out/configs.log 2>&1; echo "configs exit $?"
python -c "
import json
for l in open('gpurun_out/configs.log'):
    if l.startswith('{'): d=json.loads(l); print(d['config'], round(d['s_per_iteration'],4), d['stages_s'])"
