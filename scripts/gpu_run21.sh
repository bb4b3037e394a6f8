timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct -k regex:fce_bwd_persistent --csv --log-file gpurun_out/mask_ncu.csv python scripts/opt_ncu_probe.py "" "bwd_unit_mask=1" "bwd_unit_mask=3" "bwd_unit_mask=5" "bwd_unit_mask=6" > /dev/null 2>&1
timeout 900 python scripts/energy_probe.py --work bwd --secs 4 --sets "" "bwd_unit_mask=1" "bwd_unit_mask=3" "bwd_unit_mask=5" "bwd_unit_mask=6" "" > gpurun_out/mask_energy.log 2>&1
cat gpurun_out/mask_energy.log
