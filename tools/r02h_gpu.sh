for i in 1 2; do
  (cd abtest_old && python ../tools/scan_timing_probe.py | sed 's/^/old(CUB) /') >> gpurun_out/r02h_scan_timing.txt 2>&1
  python tools/scan_timing_probe.py | sed 's/^/new /' >> gpurun_out/r02h_scan_timing.txt 2>&1
done
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "schedule or cache or trace or acceptance or parity" > gpurun_out/r02h_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02h_tests.log
