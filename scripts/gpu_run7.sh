set -x
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/t7_all.log 2>&1; echo "rc=$?" >> gpurun_out/t7_all.log
timeout 900 python scripts/opt_probe.py "" "band_cols=3072" --blocks 8 --steps 8 > gpurun_out/ab_band3_8b.log 2>&1
timeout 900 python scripts/opt_probe.py "" "band_cols=3072" --blocks 6 --steps 3 --shape 65536,2304,256000 > gpurun_out/ab_band3_gemma.log 2>&1
timeout 900 python scripts/opt_probe.py "" "band_cols=3072" "band_cols=4096" --blocks 6 --steps 4 --shape 32768,3584,152064 > gpurun_out/ab_band3_qwen.log 2>&1
tail -2 gpurun_out/t7_all.log; grep step gpurun_out/ab_band3_*.log
