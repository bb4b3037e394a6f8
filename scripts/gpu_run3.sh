set -x
timeout 900 python scripts/energy_probe.py --work fwd --secs 4 --shape 131072,8192,128256 --sets "" "fwd_m_group=32,splits=5" "fwd_m_group=24,splits=7" "fwd_m_group=16,splits=10" "fwd_m_group=8,splits=19" > gpurun_out/fwd_raster_70b.log 2>&1
timeout 900 python scripts/energy_probe.py --work fwd --secs 3 --shape 65536,2304,256000 --sets "" "fwd_m_group=32,splits=5" "fwd_m_group=64,splits=3" "fwd_m_group=48,splits=4" "fwd_m_group=16,splits=10" > gpurun_out/fwd_raster_gemma.log 2>&1
timeout 900 python scripts/energy_probe.py --work fwd --secs 3 --shape 16384,4096,128256 --sets "" "fwd_m_group=32,splits=5" "fwd_m_group=16,splits=10" > gpurun_out/fwd_raster_8b.log 2>&1
cat gpurun_out/fwd_raster_*.log
