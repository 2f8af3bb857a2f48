# direct devShadow refresh by the exchange apply: step A/B, then the GPU suite (direct on by default)
mkdir -p gpurun_out
run() {  # tag, env...
  tag=$1; shift
  env "$@" timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --live-rounds 0 --no-cfg5 --e2e-steps 5 > /tmp/b.json 2>/dev/null
  python -c "
import json,sys;l=json.loads(open('/tmp/b.json').readline());b=l['step_breakdown_ms'];c=l['configs']
print('$tag', 'step %.4f batch %.4f va %.4f merge %.4f aborts %d cfg3 %.3f cfg4 %.3f e2e %.2f ms' % (b['step'],b['batch'],b['validate_apply'],b['merge_stage'],l['batch']['aborts_last'],c['cfg3_zipf']['ms_per_round'],c['cfg4_cache']['ms_per_round'],l['e2e']['ms_per_step']), l['bank_sum_ok'], l['shadow_equals_replica'], l['e2e']['host_replica_matches_device'])" >> gpurun_out/r02ad_sweep.txt 2>&1
}
run direct
run winner HETM_APPLY_SHADOW=0
run direct_again
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/r02ad_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02ad_tests.log
