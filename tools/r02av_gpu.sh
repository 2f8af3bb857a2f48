# cs_run_kernel (cache SCAN) occupancy variants: 4 / 5 / 6 CTAs per SM (valid-mask flags, fewer registers)
mkdir -p gpurun_out
for rep in 1 2; do for b in 4 5 6; do
  cp abvar/b$b/libhetm_b200.so paper_1905_00661_b200/libhetm_b200.so
  echo "== b$b rep$rep" >> gpurun_out/r02av_cache_variants.txt
  timeout 300 python tools/cache_sched_timeline.py 2>/dev/null | grep -E "cs_run|total" >> gpurun_out/r02av_cache_variants.txt
done; done
for b in 5 6; do
  cp abvar/b$b/libhetm_b200.so paper_1905_00661_b200/libhetm_b200.so
  timeout 900 python -m pytest tests -m gpu -x -q -k "cache" > gpurun_out/r02av_cache_tests_b$b.log 2>&1
done
