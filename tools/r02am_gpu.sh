# emit kernel: records per thread x CTAs per SM
mkdir -p gpurun_out
run() {  # tag, env...
  tag=$1; shift
  env "$@" timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --live-rounds 0 --no-configs --no-cfg5 --e2e-steps 3 > /tmp/b.json 2>/dev/null
  python -c "
import json,sys;l=json.loads(open('/tmp/b.json').readline());b=l['step_breakdown_ms']
print('$tag', 'step %.4f batch %.4f va %.4f merge %.4f e2e %.3f' % (b['step'],b['batch'],b['validate_apply'],b['merge_stage'],l['e2e']['ms_per_step']), l['bank_sum_ok'], l['shadow_equals_replica'], l['e2e']['host_replica_matches_device'])" >> gpurun_out/r02am_sweep.txt 2>&1
}
run p16_c4
run p8_c4 HETM_EMIT_PER=8
run p16_c8 HETM_EMIT_CTAS=8
run p8_c8 HETM_EMIT_PER=8 HETM_EMIT_CTAS=8
run p8_c2 HETM_EMIT_PER=8 HETM_EMIT_CTAS=2
run p16_c4_again
