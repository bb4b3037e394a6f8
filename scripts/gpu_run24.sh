timeout 900 python scripts/opt_probe.py "" "fwd_m_group=24" "splits=37" "splits=84" "fwd_m_group=24,splits=84" "fwd_m_group=40" --blocks 10 --steps 6 > gpurun_out/ab_fwd8b.log 2>&1
grep step gpurun_out/ab_fwd8b.log
