# SCAN launches of a host-buffer batch grouped in two: AUTO probe at zipf 0.5, GPU suite
mkdir -p gpurun_out
timeout 600 python tools/auto_feedback_probe.py > gpurun_out/r02al_auto_feedback.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/r02al_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02al_tests.log
