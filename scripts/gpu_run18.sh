timeout 1500 python scripts/opt_probe.py "" "fwd_m_group=16" "fwd_m_group=12" "fwd_m_group=8" --blocks 4 --steps 2 --shape 131072,8192,128256 > gpurun_out/ab_mg_70b.log 2>&1
timeout 900 python scripts/opt_probe.py "" "fwd_m_group=48" "fwd_m_group=64" "fwd_m_group=24" --blocks 6 --steps 3 --shape 65536,2304,256000 > gpurun_out/ab_mg_gemma.log 2>&1
timeout 900 python scripts/opt_probe.py "" "fwd_m_group=24" "fwd_m_group=16" --blocks 8 --steps 8 > gpurun_out/ab_mg_8b.log 2>&1
grep step gpurun_out/ab_mg_*.log
