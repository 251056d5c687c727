timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:k_mv_ -c 6 python scripts/probe_matvec.py 1 2>&1 | grep -E "k_mv_|duration|dram" | head -40
