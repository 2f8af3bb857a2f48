# A/B of the cfg2 device round on one box: the worktree build in abtest_old/ vs this tree.
ARGS="--steps 20 --warmup 5 --no-cpu-baseline --live-rounds 0 --no-configs --no-cfg5 --e2e-steps 10"
for i in 1 2 3; do
  (cd abtest_old && timeout 300 python bench.py $ARGS | grep '^{' > ../gpurun_out/ab_old_$i.json)
  timeout 300 python bench.py $ARGS | grep '^{' > gpurun_out/ab_new_$i.json
done
