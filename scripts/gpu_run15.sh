M=dram__bytes_read.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum
timeout 900 ncu --metrics $M -k regex:fce_tile_kernel --csv --log-file gpurun_out/fv_a.csv python scripts/fwd_variant_probe.py --shape 16384,8192,128256 "" "splits=37,fwd_m_group=32" > /dev/null 2>&1
timeout 900 ncu --metrics $M -k regex:fce_tile_kernel --csv --log-file gpurun_out/fv_b.csv python scripts/fwd_variant_probe.py --shape 131072,4096,128256 "" "splits=37,fwd_m_group=32" > /dev/null 2>&1
timeout 900 ncu --metrics $M -k regex:fce_tile_kernel --csv --log-file gpurun_out/fv_c.csv python scripts/fwd_variant_probe.py --shape 131072,8192,128256 "splits=37,fwd_m_group=32" "splits=74,fwd_m_group=16" > /dev/null 2>&1
echo done
