# live rounds with the pipelined merge vs the synchronous one; engine GPU tests
mkdir -p gpurun_out
for i in 1 2; do
  ./build/hetm_live_round 12 27 1048576 0 4 8 65536 1 >> gpurun_out/r02aq_live.txt 2>&1
  ./build/hetm_live_round 12 27 1048576 0 4 8 65536 0 >> gpurun_out/r02aq_live.txt 2>&1
done
timeout 1200 python -m pytest tests/test_host_engine.py tests/test_streaming.py tests/test_dispatch.py tests/test_trace_gpu.py tests/test_reports.py -m gpu -q -p no:cacheprovider > gpurun_out/r02aq_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02aq_tests.log
