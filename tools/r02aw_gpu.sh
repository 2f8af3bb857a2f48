# 2 ranks on one GPU (gloo) with the winner patch in line (HETM_WIN_SIDE=0) vs on s_win (=1);
# then the cs_run_kernel occupancy variants (4 / 5 / 6 CTAs per SM)
mkdir -p gpurun_out
cp abvar/b4/libhetm_b200.so paper_1905_00661_b200/libhetm_b200.so
export PYTHONFAULTHANDLER=1
ARGS="--gpus 2 --no-cpu-baseline --no-configs --live-rounds 0 --e2e-steps 3 --cfg5-reps 1"
for w in 0 1; do
  s=$(date +%s)
  HETM_WIN_SIDE=$w HETM_BENCH_BACKEND=gloo HETM_BENCH_ONE_GPU=1 timeout -s ABRT 360 python bench.py $ARGS \
     > gpurun_out/r02aw_2rank_win$w.json 2> gpurun_out/r02aw_2rank_win$w.err
  echo "win$w rc=$? $(( $(date +%s) - s )) s" >> gpurun_out/r02aw_2rank.txt
done
for rep in 1 2; do for b in 4 5 6; do
  cp abvar/b$b/libhetm_b200.so paper_1905_00661_b200/libhetm_b200.so
  echo "== b$b rep$rep" >> gpurun_out/r02av_cache_variants.txt
  timeout 300 python tools/cache_sched_timeline.py 2>/dev/null | grep -E "cs_run|total" >> gpurun_out/r02av_cache_variants.txt
done; done
for b in 5 6; do
  cp abvar/b$b/libhetm_b200.so paper_1905_00661_b200/libhetm_b200.so
  timeout 600 python -m pytest tests -m gpu -x -q -k "cache" > gpurun_out/r02av_cache_tests_b$b.log 2>&1
done
