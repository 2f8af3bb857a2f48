# stripe kernel after prefetch / release-before-RED / sit-out: CTAs-per-SM x table sweep, then the GPU suite
mkdir -p gpurun_out
run() {  # tag, env...
  tag=$1; shift
  env "$@" timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --live-rounds 0 --no-configs --no-cfg5 --e2e-steps 3 > /tmp/b.json 2>/dev/null
  python -c "
import json,sys;l=json.loads(open('/tmp/b.json').readline());b=l['step_breakdown_ms']
print('$tag', 'step %.4f batch %.4f va %.4f merge %.4f aborts %d' % (b['step'],b['batch'],b['validate_apply'],b['merge_stage'],l['batch']['aborts_last']), l['bank_sum_ok'], l['shadow_equals_replica'])" >> gpurun_out/r02p_sweep.txt 2>&1
}
for bits in 22 23; do for b in 1 2 3 4; do
  run bits${bits}_b${b} HETM_STRIPE_BITS=$bits HETM_TX_BLOCKS_PER_SM=$b
done; done
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/r02p_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02p_tests.log
