timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_fuzz_gpu.py -x -q -m gpu > gpurun_out/t31.log 2>&1; echo "rc=$?" >> gpurun_out/t31.log
timeout 900 python scripts/opt_probe.py "" "bwd_unit_mask=263" --blocks 16 --steps 8 > gpurun_out/ab_dbuf.log 2>&1
timeout 900 python scripts/opt_probe.py "" "bwd_unit_mask=263" --blocks 6 --steps 3 --shape 65536,2304,256000 > gpurun_out/ab_dbuf_gemma.log 2>&1
tail -n 2 gpurun_out/t31.log; grep step gpurun_out/ab_dbuf*.log
