timeout 1500 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:"k_seg_tn|k_ml_proj|k_ml_update|k_proj_cat|k_leafid" --csv --log-file gpurun_out/traffic.csv python scripts/one_step.py 20 > gpurun_out/ncu_traffic.log 2>&1; echo "ncu exit $?"
tail -3 gpurun_out/ncu_traffic.log
