timeout 900 python scripts/opt_probe.py "" "bwd_epi_warps=4" "l2_hints=9" "l2_hints=0" "l2_hints=3" --blocks 10 --steps 6 > gpurun_out/ab_misc.log 2>&1
grep step gpurun_out/ab_misc.log
