timeout 900 python scripts/opt_probe.py "" "bwd_unit_mask=1031" "bwd_unit_mask=2055" "bwd_unit_mask=3591" --blocks 12 --steps 6 > gpurun_out/ab_pace.log 2>&1
grep step gpurun_out/ab_pace.log
