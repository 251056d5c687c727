nproc; lscpu | grep "Model name"; grep MemTotal /proc/meminfo
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 2400 python scripts/diag_c4.py 14 16 17 18 20 --cpu-max=16 > gpurun_out/diag_c4.log 2>&1
echo rc=$?
