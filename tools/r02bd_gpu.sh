# after the pre-roll fix: the 2-rank bench 12x (was hanging ~1 in 5-7), the GPU suite, the N=1 bench
mkdir -p gpurun_out
export PYTHONFAULTHANDLER=1
for i in $(seq 1 12); do
  s=$(date +%s)
  HETM_BENCH_BACKEND=gloo HETM_BENCH_ONE_GPU=1 timeout -s KILL 120 python bench.py --steps 3 --warmup 3 --gpus 2 --no-cpu-baseline --no-configs --live-rounds 0 --e2e-steps 3 --cfg5-reps 1 > gpurun_out/r02bd_run$i.out 2> gpurun_out/r02bd_run$i.err
  echo "run$i rc=$? $(( $(date +%s) - s )) s" >> gpurun_out/r02bd_runs.txt
done
s=$(date +%s); timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r02bd_gpu_tests.log 2>&1; echo "rc=$? $(( $(date +%s) - s )) s" >> gpurun_out/r02bd_gpu_tests.log
timeout 600 python bench.py > gpurun_out/r02bd_bench_n1.json 2> gpurun_out/r02bd_bench_n1.err
