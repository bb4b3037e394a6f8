timeout 900 python bench.py --gpus 8 --steps 5 --warmup 3 --no-e2e-grads > gpurun_out/b8_local.json 2> gpurun_out/b8_local.err; echo "rc=$?" >> gpurun_out/b8_local.err
timeout 1200 python bench.py --gpus 4 --transport ipc --steps 5 --warmup 3 --no-e2e-grads > gpurun_out/b4_ipc.json 2> gpurun_out/b4_ipc.err; echo "rc=$?" >> gpurun_out/b4_ipc.err
tail -n 2 gpurun_out/b8_local.err gpurun_out/b4_ipc.err
