# Generic GPU-box wrapper: build in place, then run the given command with its
# output in gpurun_out/<tag>.log.  Usage: bash scripts/gpu_run.sh <tag> <cmd...>
tag=$1; shift
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$tag.log 2>&1 || { echo build failed; tail -20 gpurun_out/build_$tag.log; exit 1; }
"$@" > gpurun_out/$tag.log 2>&1
rc=$?
echo "rc=$rc"; tail -5 gpurun_out/$tag.log
exit $rc
