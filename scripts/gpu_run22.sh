timeout 900 python scripts/energy_probe.py --work fwd,bwd --secs 4 --sets "bwd_unit_mask=1" "bwd_unit_mask=1,bwd_tma_epi=2" "bwd_unit_mask=9,bwd_tma_epi=2" "bwd_unit_mask=1" > gpurun_out/mask2_energy.log 2>&1
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed -k regex:fce_bwd_persistent --csv --log-file gpurun_out/mask2_ncu.csv python scripts/opt_ncu_probe.py "bwd_unit_mask=1" "bwd_unit_mask=9,bwd_tma_epi=2" > /dev/null 2>&1
cat gpurun_out/mask2_energy.log
