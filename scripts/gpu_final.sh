set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench exit $?"
cat gpurun_out/bench.json
timeout 900 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref exit $?"
cat gpurun_out/bench_ref.json
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python scripts/one_step.py 20 > gpurun_out/ncu_launch.log 2>&1; echo "ncu exit $?"
python scripts/launch_summary.py gpurun_out/launches.csv > gpurun_out/launch_summary.md
timeout 900 ncu --set full --import-source on --kernel-name-base demangled -k "regex:k_seg_tn<.int.80, .int.80>" --launch-skip 40 -c 1 -o gpurun_out/segtn8080 python scripts/one_step.py 20 > gpurun_out/ncu_full.log 2>&1; echo "ncu full exit $?"
timeout 900 python scripts/bench_configs.py 3 > gpurun_out/configs.log 2>&1; echo "configs exit $?"; tail -8 gpurun_out/configs.log
