timeout 900 python scripts/opt_probe.py "" "bwd_epi_warps=4" --blocks 16 --steps 8 > gpurun_out/ab_epi.log 2>&1
timeout 900 python scripts/energy_probe.py --work bwd --secs 4 --sets "" "bwd_epi_warps=4" "" "bwd_epi_warps=4" > gpurun_out/epi_energy.log 2>&1
timeout 900 python scripts/opt_probe.py "" "bwd_epi_warps=4" --blocks 6 --steps 3 --shape 65536,2304,256000 > gpurun_out/ab_epi_gemma.log 2>&1
timeout 900 python scripts/opt_probe.py "" "bwd_epi_warps=4" --blocks 4 --steps 2 --shape 131072,8192,128256 > gpurun_out/ab_epi_70b.log 2>&1
grep step gpurun_out/ab_epi*.log; cat gpurun_out/epi_energy.log
