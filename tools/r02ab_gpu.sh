mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/r02ab_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02ab_tests.log
