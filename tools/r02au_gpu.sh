# A/B: devShadow winner patch on a side stream (HETM_WIN_SIDE=1, product) vs in line on s_merge
mkdir -p gpurun_out
ARGS="--steps 20 --warmup 5 --no-cpu-baseline --live-rounds 0 --no-configs --no-cfg5 --e2e-steps 10"
for i in 1 2 3; do
  HETM_WIN_SIDE=0 timeout 300 python bench.py $ARGS 2>/dev/null | grep '^{' > gpurun_out/r02au_inline_$i.json
  HETM_WIN_SIDE=1 timeout 300 python bench.py $ARGS 2>/dev/null | grep '^{' > gpurun_out/r02au_side_$i.json
done
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02au_gpu_tests.log 2>&1
