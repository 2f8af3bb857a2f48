timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/r02f_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02f_tests.log
timeout 900 python tools/ncu_all.py > gpurun_out/r02f_ncu_all_plain.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -o gpurun_out/r02f_all python tools/ncu_all.py > gpurun_out/r02f_ncu_all.log 2>&1
