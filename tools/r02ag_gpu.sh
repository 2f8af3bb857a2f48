mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_stripe_sharing.py -m gpu -q -p no:cacheprovider > gpurun_out/r02ag_sharing_test.log 2>&1; echo "rc=$?" >> gpurun_out/r02ag_sharing_test.log
run() {  # tag, env...
  tag=$1; shift
  env "$@" timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --live-rounds 0 --no-configs --no-cfg5 --e2e-steps 3 > /tmp/b.json 2>/dev/null
  python -c "
import json,sys;l=json.loads(open('/tmp/b.json').readline());b=l['step_breakdown_ms']
print('$tag', 'step %.4f batch %.4f va %.4f merge %.4f aborts %d' % (b['step'],b['batch'],b['validate_apply'],b['merge_stage'],l['batch']['aborts_last']), l['bank_sum_ok'], l['shadow_equals_replica'])" >> gpurun_out/r02ag_sweep.txt 2>&1
}
run b24
run b23 HETM_STRIPE_BITS=23
run b22 HETM_STRIPE_BITS=22
run b24_again
run b23_again HETM_STRIPE_BITS=23
HETM_STRIPE_BITS=23 timeout 600 python tools/stripe_skew_probe.py > gpurun_out/r02ag_skew23.txt 2>&1
