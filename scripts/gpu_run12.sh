timeout 900 python -m pytest tests/test_multirank_gpu.py -x -q -k random > gpurun_out/t12.log 2>&1; echo "rc=$?" >> gpurun_out/t12.log
tail -n 5 gpurun_out/t12.log
