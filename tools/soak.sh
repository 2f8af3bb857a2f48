# Soak run (not part of the test suite): longer live rounds through the checker
# and the oracle, to catch rare races.  bash tools/soak.sh > gpurun_out/soak.txt
set -u
for pol in host device; do
  build/trace_test 30 0 0 "" $pol | tail -1
done
build/round_test 40 20 16384 4 3 host 3 3 1 | tail -1
build/round_test 40 20 16384 4 3 device 3 2 1 | tail -1
build/queue_round_test 20 4096 | tail -1
for k in 1 2; do python -m pytest tests/test_acceptance.py -q -m gpu -p no:cacheprovider 2>&1 | tail -1; done
