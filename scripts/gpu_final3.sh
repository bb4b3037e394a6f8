set -x
TAG=r02f bash scripts/gpu_configs.sh
timeout 1800 python -m pytest tests -x -q -m gpu > gpurun_out/final_tests.log 2>&1; echo "rc=$?" >> gpurun_out/final_tests.log
tail -n 3 gpurun_out/final_tests.log
