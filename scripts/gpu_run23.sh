timeout 900 python scripts/opt_probe.py "" "l2_hints=17" "l2_hints=16" "l2_hints=3" --blocks 8 --steps 8 > gpurun_out/ab_hints.log 2>&1
timeout 900 python scripts/energy_probe.py --work bwd --secs 4 --sets "" "l2_hints=17" "" "l2_hints=17" > gpurun_out/hints_energy.log 2>&1
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:fce_bwd_persistent --csv --log-file gpurun_out/hints_ncu.csv python scripts/opt_ncu_probe.py "" "l2_hints=17" > /dev/null 2>&1
grep step gpurun_out/ab_hints.log; cat gpurun_out/hints_energy.log
