timeout 900 python scripts/opt_probe.py "" "bwd_tma_epi=1" "bwd_tma_epi=2" "splits=84" --blocks 10 --steps 6 > gpurun_out/ab_tmaepi.log 2>&1
grep step gpurun_out/ab_tmaepi.log
