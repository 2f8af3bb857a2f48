# host-fed apply form: validate tests, step + cfg3 sweep, GPU suite; then (EXPERIMENTS build) stripe knockouts
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -x -k "validate" > gpurun_out/r02u_validate_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02u_validate_tests.log
run() {  # tag, env...
  tag=$1; shift
  env "$@" timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --live-rounds 0 --no-cfg5 --e2e-steps 3 > /tmp/b.json 2>/dev/null
  python -c "
import json,sys;l=json.loads(open('/tmp/b.json').readline());b=l['step_breakdown_ms'];c=l['configs']
print('$tag', 'step %.4f batch %.4f va %.4f merge %.4f aborts %d cfg3 %.3f ms cfg4 %.3f ms' % (b['step'],b['batch'],b['validate_apply'],b['merge_stage'],l['batch']['aborts_last'],c['cfg3_zipf']['ms_per_round'],c['cfg4_cache']['ms_per_round']), l['bank_sum_ok'], l['shadow_equals_replica'])" >> gpurun_out/r02u_sweep.txt 2>&1
}
run hostfed
run amax HETM_APPLY_AMAX=1
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/r02u_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02u_tests.log
bash tools/r02t_gpu.sh
