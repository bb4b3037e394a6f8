set -x
export FCE_LOCAL_TIMEOUT_S=1200
timeout 1500 compute-sanitizer --tool memcheck --leak-check no --error-exitcode 9 python -m pytest tests/test_multirank_gpu.py -x -q -k "match_oracle and (2-sum or 3-mean) or overlapped and (2-2 or 3-3) or sp_gather_and or dp_step_matches or collectives" > gpurun_out/san_memcheck.log 2>&1; echo "memcheck rc=$?" >> gpurun_out/san_memcheck.log
timeout 1500 compute-sanitizer --tool racecheck --error-exitcode 9 python -m pytest tests/test_multirank_gpu.py -x -q -k "collectives" > gpurun_out/san_racecheck.log 2>&1; echo "racecheck rc=$?" >> gpurun_out/san_racecheck.log
tail -5 gpurun_out/san_memcheck.log gpurun_out/san_racecheck.log
