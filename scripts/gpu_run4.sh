set -x
timeout 900 python scripts/energy_probe.py --work bwd --secs 3 --shape 65536,2304,256000 --sets "" "band_cols=6144" "band_cols=12288" "row_chunk=32768,band_cols=6144" > gpurun_out/band_gemma.log 2>&1
timeout 900 python scripts/energy_probe.py --work bwd --secs 3 --shape 32768,3584,152064 --ignore 0.25 --sets "" "band_cols=6144" "band_cols=12288" > gpurun_out/band_qwen.log 2>&1
timeout 900 python scripts/energy_probe.py --work bwd --secs 3 --shape 16384,4096,128256 --sets "" "band_cols=6144" "band_cols=12288" "band_cols=4096" > gpurun_out/band_8b.log 2>&1
timeout 900 python scripts/energy_probe.py --work bwd --secs 4 --shape 131072,8192,128256 --sets "" "band_cols=6144" "row_chunk=131072,band_cols=3072" > gpurun_out/band_70b.log 2>&1
cat gpurun_out/band_*.log
