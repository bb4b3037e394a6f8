set -x
timeout 900 python scripts/opt_probe.py "" "band_cols=3584" "band_cols=3840" "band_cols=4096" "band_cols=4608" "band_cols=5120" --blocks 8 --steps 8 > gpurun_out/ab_band2_8b.log 2>&1
timeout 900 python scripts/opt_probe.py "" "band_cols=3584" "band_cols=4096" "band_cols=5120" --blocks 6 --steps 3 --shape 65536,2304,256000 > gpurun_out/ab_band2_gemma.log 2>&1
timeout 900 python scripts/opt_probe.py "" "band_cols=3584" "band_cols=4096" --blocks 4 --steps 2 --shape 131072,8192,128256 > gpurun_out/ab_band2_70b.log 2>&1
grep step gpurun_out/ab_band2_*.log
