timeout 900 python -m pytest tests/test_multirank_gpu.py tests/test_bench.py -x -q -m gpu -k "ipc" > gpurun_out/t13.log 2>&1; echo "rc=$?" >> gpurun_out/t13.log
tail -n 30 gpurun_out/t13.log
