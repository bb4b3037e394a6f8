timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:fce_bwd_persistent --csv --log-file gpurun_out/dhg_ncu.csv python scripts/g_residency_probe.py --geoms 0:0:1:1,0:0:1:2 > /dev/null 2>&1
timeout 900 python scripts/energy_probe.py --work bwd,copy --secs 4 --sets "" "dh_group=2" "" "dh_group=2" > gpurun_out/dhg_energy.log 2>&1
cat gpurun_out/dhg_energy.log
