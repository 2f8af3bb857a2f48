python tools/scan_timing_probe.py | sed 's/^/new /' >> gpurun_out/r02i_scan_timing.txt 2>&1
(cd abtest_old && python ../tools/scan_timing_probe.py | sed 's/^/old(CUB) /') >> gpurun_out/r02i_scan_timing.txt 2>&1
python tools/scan_timing_probe.py | sed 's/^/new /' >> gpurun_out/r02i_scan_timing.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "schedule or cache or acceptance" > gpurun_out/r02i_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02i_tests.log
