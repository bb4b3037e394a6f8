( time timeout 1800 python bench.py --gpus 1 --steps 20 --warmup 5 ) > gpurun_out/dl2_n1.json 2> gpurun_out/dl2_n1.err
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/dl2_smoke.log 2>&1
tail -n 4 gpurun_out/dl2_n1.err; cat gpurun_out/dl2_smoke.log
