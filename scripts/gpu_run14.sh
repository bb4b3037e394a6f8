timeout 1200 python -m pytest tests/test_multirank_gpu.py -x -q -k "fused or sp_vp or ipc" > gpurun_out/t14.log 2>&1; echo "rc=$?" >> gpurun_out/t14.log
tail -n 40 gpurun_out/t14.log
