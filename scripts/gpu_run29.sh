timeout 900 python scripts/opt_probe.py "" "band_cols=4096" "band_cols=3072" "band_cols=4608" --blocks 10 --steps 6 > gpurun_out/ab_band4.log 2>&1
timeout 900 python scripts/opt_probe.py "" "band_cols=3584" "band_cols=5120" --blocks 6 --steps 3 --shape 65536,2304,256000 > gpurun_out/ab_band4_gemma.log 2>&1
grep step gpurun_out/ab_band4*.log
