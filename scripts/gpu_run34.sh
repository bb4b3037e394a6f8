for v in 128256 64128 32064 16032; do
  timeout 600 python scripts/opt_probe.py "" --blocks 6 --steps 6 --shape 16384,4096,$v 2>&1 | grep step | sed "s/^/V=$v /"
done > gpurun_out/shard_shapes.log
cat gpurun_out/shard_shapes.log
