set -x
timeout 900 python -m pytest tests/test_gpu_hmatvec.py tests/test_gpu_hodlr.py tests/test_gpu_c4_properties.py -x -q > gpurun_out/pytest_mv.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_mv.log
tail -5 gpurun_out/pytest_mv.log
timeout 600 python scripts/probe_matvec.py > gpurun_out/probe_mv.log 2>&1; cat gpurun_out/probe_mv.log
timeout 900 ncu --set full --import-source on -k regex:k_mv_ -c 2 -o gpurun_out/mv_full python scripts/probe_matvec.py 1 > gpurun_out/ncu_mv.log 2>&1; echo "ncu exit $?"; tail -3 gpurun_out/ncu_mv.log
