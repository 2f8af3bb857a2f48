# merge stage: one counter memset, record-count copy off s_merge: step sweep + GPU suite + timeline
mkdir -p gpurun_out
run() {  # tag, env...
  tag=$1; shift
  env "$@" timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --live-rounds 0 --no-configs --no-cfg5 --e2e-steps 3 > /tmp/b.json 2>/dev/null
  python -c "
import json,sys;l=json.loads(open('/tmp/b.json').readline());b=l['step_breakdown_ms']
print('$tag', 'step %.4f batch %.4f va %.4f merge %.4f aborts %d' % (b['step'],b['batch'],b['validate_apply'],b['merge_stage'],l['batch']['aborts_last']), l['bank_sum_ok'], l['shadow_equals_replica'], l['e2e']['host_replica_matches_device'])" >> gpurun_out/r02ai_sweep.txt 2>&1
}
run a
run b
run c
timeout 300 python tools/bench_step_timeline.py > gpurun_out/r02ai_step_timeline.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/r02ai_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02ai_tests.log
