mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_bank_schedule.py -m gpu -q -p no:cacheprovider > gpurun_out/r02aa_sched_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02aa_sched_tests.log
timeout 600 python tools/auto_feedback_probe.py > gpurun_out/r02aa_auto_feedback.txt 2>&1
timeout 600 python tools/stripe_skew_probe.py > gpurun_out/r02aa_skew.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/r02aa_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02aa_tests.log
