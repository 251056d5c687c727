# GPU-box job: build in place, then run each "tag|timeout|command" line of the
# job file given as $1, logging to gpurun_out/<tag>.log.
# Usage: bash scripts/gpu_job.sh jobs.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; tail -20 gpurun_out/build.log; exit 1; }
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
nproc >> gpurun_out/gpu.txt; lscpu | grep 'Model name' >> gpurun_out/gpu.txt
while IFS='|' read -r tag to cmd; do
  [ -z "$tag" ] && continue
  case "$tag" in \#*) continue;; esac
  t0=$(date +%s)
  timeout "$to" bash -c "$cmd" > "gpurun_out/$tag.log" 2>&1
  echo "$tag rc=$? $(( $(date +%s) - t0 ))s"
done < "$1"
