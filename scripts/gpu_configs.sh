# Per-config bench lines + ncu launch list + ncu --set full of the step (round 2).
set -x
TAG=${TAG:-r02}
for c in ${CONFIGS:-llama3-8b qwen2.5-7b gemma2-2b llama3-70b}; do
  extra="--no-cpu-baseline --no-dropin"
  [ "$c" = "llama3-8b" ] && extra=""
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 $extra > gpurun_out/${TAG}_bench_$c.json 2> gpurun_out/${TAG}_bench_$c.err
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
      --log-file gpurun_out/${TAG}_${c}_launches.csv python scripts/profile_step.py --config $c > /dev/null 2>&1
  timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off \
      -k regex:"fce_bwd_persistent|fce_tile_kernel" -f -o gpurun_out/${TAG}_${c}_full \
      python scripts/profile_step.py --config $c > gpurun_out/${TAG}_${c}_ncu.log 2>&1
done
ls -la gpurun_out/
