set -x
timeout 900 python scripts/opt_probe.py "" "band_cols=4096" "band_cols=3584" --blocks 8 --steps 8 > gpurun_out/ab_band_8b.log 2>&1
timeout 900 python scripts/opt_probe.py "" "band_cols=4096" "band_cols=6144" --blocks 6 --steps 3 --shape 65536,2304,256000 > gpurun_out/ab_band_gemma.log 2>&1
timeout 900 python scripts/opt_probe.py "" "band_cols=4096" --blocks 6 --steps 4 --shape 32768,3584,152064 > gpurun_out/ab_band_qwen.log 2>&1
cat gpurun_out/ab_band_*.log
