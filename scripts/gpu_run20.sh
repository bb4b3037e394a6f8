export FCE_LOCAL_TIMEOUT_S=1200
timeout 2400 compute-sanitizer --tool memcheck --leak-check no --error-exitcode 9 python -m pytest tests/test_multirank_gpu.py -x -q -k "fused_dh_reduction and 2-mean or sp_vp_backward_reduce and 3-None or overlapped and 2-2 or fallbacks" > gpurun_out/san2_memcheck.log 2>&1; echo "memcheck rc=$?" >> gpurun_out/san2_memcheck.log
timeout 2400 compute-sanitizer --tool synccheck --error-exitcode 9 python -m pytest tests/test_multirank_gpu.py -x -q -k "fused_dh_reduction and 2-mean or collectives" > gpurun_out/san2_synccheck.log 2>&1; echo "synccheck rc=$?" >> gpurun_out/san2_synccheck.log
tail -n 4 gpurun_out/san2_memcheck.log gpurun_out/san2_synccheck.log
