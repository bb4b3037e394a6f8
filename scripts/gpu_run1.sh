set -x
nvidia-smi --query-gpu=name,clocks.sm,power.draw --format=csv
timeout 900 python -m pytest tests/test_multirank_gpu.py tests/test_torch_op_gpu.py tests/test_bench.py tests/test_dropin_cpp.py -x -q -m gpu > gpurun_out/t_new.log 2>&1; echo "new rc=$?" >> gpurun_out/t_new.log
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/t_all.log 2>&1; echo "all rc=$?" >> gpurun_out/t_all.log
timeout 600 python bench.py > gpurun_out/bench1.json 2> gpurun_out/bench1.err; echo "bench rc=$?" >> gpurun_out/bench1.err
tail -3 gpurun_out/t_new.log gpurun_out/t_all.log; cat gpurun_out/bench1.json | head -c 3000
