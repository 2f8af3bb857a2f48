# stripe table size / P0 spin / CTAs per SM sweep of the bench step; exchange apply vs atomicMax apply
mkdir -p gpurun_out
./build/stripe_probe 2>&1 | grep -E "apply" > gpurun_out/r02n_apply_probe.txt
run() {  # tag, env...
  tag=$1; shift
  env "$@" timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --live-rounds 0 --no-configs --no-cfg5 --e2e-steps 3 > /tmp/b.json 2>/dev/null
  python -c "
import json,sys;l=json.loads(open('/tmp/b.json').readline());b=l['step_breakdown_ms']
print('$tag', 'step %.4f batch %.4f va %.4f merge %.4f aborts %d' % (b['step'],b['batch'],b['validate_apply'],b['merge_stage'],l['batch']['aborts_last']), l['bank_sum_ok'], l['shadow_equals_replica'])" >> gpurun_out/r02n_sweep.txt 2>&1
}
run amax_b2_s22 HETM_APPLY_AMAX=1 HETM_TX_BLOCKS_PER_SM=2
for bits in 22 23 24; do for spin in 0 1; do for b in 1 2; do
  run bits${bits}_spin${spin}_b${b} HETM_STRIPE_BITS=$bits HETM_STRIPE_SPIN=$spin HETM_TX_BLOCKS_PER_SM=$b
done; done; done
