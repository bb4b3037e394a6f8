# What the driver runs at round end, in order (reference arm first).
set -x
( time timeout 1800 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 ) > gpurun_out/dl_ref.json 2> gpurun_out/dl_ref.err
( time timeout 1800 python bench.py --gpus 1 --steps 20 --warmup 5 ) > gpurun_out/dl_n1.json 2> gpurun_out/dl_n1.err
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/dl_smoke.log 2>&1
tail -n 4 gpurun_out/dl_ref.err gpurun_out/dl_n1.err; cat gpurun_out/dl_smoke.log
