# usage: ncu_to_md.sh <name> <ncu args...> -- <command...>
# Runs one `ncu --set full` capture into gpurun_out/<name>.ncu-rep, writes the
# summary (scripts/ncu_summary.py) to gpurun_out/<name>.txt and deletes the
# report (gpurun copies back at most 64 MiB).
name=$1; shift
args=(); while [ "$1" != "--" ]; do args+=("$1"); shift; done; shift
ncu --set full --clock-control none --import-source on "${args[@]}" -o gpurun_out/$name -f "$@" > gpurun_out/$name.log 2>&1
python scripts/ncu_summary.py gpurun_out/$name.ncu-rep > gpurun_out/$name.txt 2>&1
ls -la gpurun_out/$name.ncu-rep >> gpurun_out/$name.log
rm -f gpurun_out/$name.ncu-rep
