set -x
timeout 900 python scripts/opt_probe.py "" "dh_group=2" "dh_group=3" "dh_group=2,band_cols=3072" --blocks 8 --steps 6 > gpurun_out/ab_dhg_8b.log 2>&1
timeout 900 python scripts/opt_probe.py "" "dh_group=2" --blocks 4 --steps 2 --shape 65536,2304,256000 > gpurun_out/ab_dhg_gemma.log 2>&1
grep step gpurun_out/ab_dhg_*.log
