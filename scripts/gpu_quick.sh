timeout 300 python scripts/probe_matvec.py 64 2>&1 | grep "s=64"
timeout 600 python scripts/one_step.py 20 2>&1 | tail -1
timeout 600 python -m pytest tests/test_gpu_hodlr.py tests/test_gpu_hmatvec.py tests/test_gpu_factor_trace.py -q 2>&1 | tail -1
