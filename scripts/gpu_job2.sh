python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_job2.log 2>&1 || { tail -20 gpurun_out/build_job2.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_dropin.py tests/test_gpu_acceptance.py -q -x > gpurun_out/pytest_new.log 2>&1; echo "pytest rc=$?"
timeout 600 python scripts/probe_parity_modes.py 4096 > gpurun_out/parity_modes.log 2>&1; echo "modes rc=$?"
timeout 1500 python scripts/diag_levels2.py 17 18 --cpu=18 > gpurun_out/diag_levels2.log 2>&1; echo "levels2 rc=$?"
