set -x
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "merge or parity or acceptance or cfg5 or shadow or rollback or streaming or engine" > gpurun_out/r02d_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02d_tests.log
for w in 40 32 31 30; do for ab in 31; do
  HETM_APPLY_WINDOW_LOG2=$w HETM_APPLY_WINDOW_ABOVE_LOG2=$ab timeout 300 python tools/bucket_apply_probe.py 32 33 2>&1 | grep "B=  1" | sed "s/^/win=$w above=$ab /" >> gpurun_out/r02d_window_probe.txt
done; done
timeout 600 python bench.py --steps 10 --warmup 5 --no-cpu-baseline --live-rounds 0 --no-configs > gpurun_out/r02d_bench.log 2>&1
