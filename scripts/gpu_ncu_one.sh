# usage: bash scripts/gpu_ncu_one.sh <kernel-regex> <launch-skip> <name>
timeout 900 ncu --set full --import-source on --kernel-name-base demangled -k "regex:$1" --launch-skip $2 -c 1 -o gpurun_out/$3 python scripts/one_step.py 20 > gpurun_out/ncu_$3.log 2>&1; echo "ncu exit $?"
