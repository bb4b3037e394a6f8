timeout 900 python scripts/opt_probe.py "" "bwd_reserve_sms=4" "bwd_reserve_sms=8" "bwd_reserve_sms=16" --blocks 10 --steps 6 > gpurun_out/ab_reserve.log 2>&1
grep step gpurun_out/ab_reserve.log
