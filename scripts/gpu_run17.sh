M=dram__bytes_read.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum
timeout 1500 ncu --metrics $M -k regex:fce_tile_kernel --csv --log-file gpurun_out/fv_d.csv python scripts/fwd_variant_probe.py --shape 131072,8192,128256 "" "fwd_m_group=16" "fwd_m_group=24" "fwd_m_group=48" "fwd_m_group=64" "splits=84" "splits=251" "fwd_m_group=16,splits=251" > /dev/null 2>&1
echo done
