timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python scripts/one_step.py 20 > gpurun_out/ncu_launch.log 2>&1; echo "ncu exit $?"
python scripts/launch_summary.py gpurun_out/launches.csv > gpurun_out/launch_summary.md; head -60 gpurun_out/launch_summary.md
