mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_host_engine.py tests/test_streaming.py -m gpu -q -p no:cacheprovider > gpurun_out/r02ar_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02ar_tests.log
