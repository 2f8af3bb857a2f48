# intermittent hang of the 2-ranks-on-one-GPU bench (test_two_ranks_on_one_gpu): the tests that run
# before it in the suite, then the same command 5x with Python stack dumps on timeout (SIGABRT)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_acceptance.py tests/test_bank_schedule.py -m gpu -x -q > gpurun_out/r02bb_pre.log 2>&1
export PYTHONFAULTHANDLER=1 HETM_BENCH_BACKEND=gloo HETM_BENCH_ONE_GPU=1
for i in 1 2 3 4 5; do
  s=$(date +%s)
  timeout -s ABRT 150 python bench.py --steps 3 --warmup 3 --gpus 2 --no-cpu-baseline --no-configs --live-rounds 0 --e2e-steps 3 --cfg5-reps 1 > gpurun_out/r02bb_run$i.out 2> gpurun_out/r02bb_run$i.err
  echo "run$i rc=$? $(( $(date +%s) - s )) s" >> gpurun_out/r02bb_runs.txt
  nvidia-smi --query-compute-apps=pid,used_memory --format=csv >> gpurun_out/r02bb_runs.txt 2>&1
done
