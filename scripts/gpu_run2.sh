set -x
nvidia-smi --query-gpu=name,clocks.sm,power.draw --format=csv
timeout 900 python -m pytest tests/test_multirank_gpu.py tests/test_cli.py tests/test_torch_op_gpu.py -x -q -m gpu > gpurun_out/t2_new.log 2>&1; echo "rc=$?" >> gpurun_out/t2_new.log
timeout 600 python -m pytest tests/test_parity_gpu.py -x -q -m gpu -k "sentinel or zero_hidden" >> gpurun_out/t2_new.log 2>&1; echo "rc=$?" >> gpurun_out/t2_new.log
timeout 300 python scripts/vp_overlap_trace.py > gpurun_out/overlap_trace.log 2>&1
timeout 300 python scripts/vp_overlap_trace.py --chunks 4 --reserve 8 >> gpurun_out/overlap_trace.log 2>&1
timeout 600 python scripts/energy_probe.py --work bwd --secs 3 --sets "" "row_chunk=4096,band_cols=3072" "row_chunk=8192,band_cols=1536" "row_chunk=2048,band_cols=6144" "row_chunk=16384,band_cols=768" > gpurun_out/g_energy.log 2>&1
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:fce_bwd_persistent --csv --log-file gpurun_out/g_ncu.csv python scripts/g_residency_probe.py > gpurun_out/g_probe.log 2>&1
tail -3 gpurun_out/t2_new.log; cat gpurun_out/overlap_trace.log gpurun_out/g_energy.log gpurun_out/g_probe.log
