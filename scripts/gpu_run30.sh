timeout 900 python scripts/opt_probe.py "" "fwd_pair=1" "fwd_mc=1" "fwd_pair=1,fwd_m_group=16" --blocks 10 --steps 6 > gpurun_out/ab_fwdvar.log 2>&1
grep step gpurun_out/ab_fwdvar.log
