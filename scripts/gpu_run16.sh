M=dram__bytes_read.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum
timeout 900 ncu --metrics $M -k regex:fce_tile_kernel --csv --log-file gpurun_out/pad_a.csv python scripts/ld_pad_probe.py --shape 16384,8192,128256 --pads 0,64,8 > /dev/null 2>&1
timeout 900 ncu --metrics $M -k regex:fce_tile_kernel --csv --log-file gpurun_out/pad_c.csv python scripts/ld_pad_probe.py --shape 131072,8192,128256 --pads 0,64 > /dev/null 2>&1
timeout 900 ncu --metrics $M -k regex:fce_tile_kernel --csv --log-file gpurun_out/pad_b.csv python scripts/ld_pad_probe.py --shape 16384,4096,128256 --pads 0,64 > /dev/null 2>&1
echo done
