set -x
timeout 900 python bench.py > gpurun_out/b11_n1.json 2> gpurun_out/b11_n1.err; echo "rc=$?" >> gpurun_out/b11_n1.err
timeout 900 python bench.py --gpus 2 --steps 5 --no-e2e-grads > gpurun_out/b11_n2.json 2> gpurun_out/b11_n2.err; echo "rc=$?" >> gpurun_out/b11_n2.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/b11_ref.json 2> gpurun_out/b11_ref.err; echo "rc=$?" >> gpurun_out/b11_ref.err
cat gpurun_out/b11_n1.json gpurun_out/b11_n2.json gpurun_out/b11_ref.json; tail -n 3 gpurun_out/b11_*.err
