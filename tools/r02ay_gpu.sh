# A/B: stripe table in a persisting L2 carve-out (HETM_L2_PERSIST=1) vs plain
mkdir -p gpurun_out
ARGS="--steps 20 --warmup 5 --no-cpu-baseline --live-rounds 0 --no-configs --no-cfg5 --e2e-steps 10"
for i in 1 2 3; do
  HETM_L2_PERSIST=0 timeout 300 python bench.py $ARGS 2>/dev/null | grep '^{' > gpurun_out/r02ay_plain_$i.json
  HETM_L2_PERSIST=1 timeout 300 python bench.py $ARGS 2>gpurun_out/r02ay_persist_$i.err | grep '^{' > gpurun_out/r02ay_persist_$i.json
done
