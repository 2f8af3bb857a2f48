# P1-after-P2 stripe kernel + CAS put-back apply: quick step sweep, GPU suite, full bench, ncu of every product kernel
mkdir -p gpurun_out
run() {  # tag, env...
  tag=$1; shift
  env "$@" timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --live-rounds 0 --no-cfg5 --e2e-steps 3 > /tmp/b.json 2>/dev/null
  python -c "
import json,sys;l=json.loads(open('/tmp/b.json').readline());b=l['step_breakdown_ms'];c=l['configs']
print('$tag', 'step %.4f batch %.4f va %.4f merge %.4f aborts %d cfg3 %.3f ms cfg4 %.3f ms' % (b['step'],b['batch'],b['validate_apply'],b['merge_stage'],l['batch']['aborts_last'],c['cfg3_zipf']['ms_per_round'],c['cfg4_cache']['ms_per_round']), l['bank_sum_ok'], l['shadow_equals_replica'])" >> gpurun_out/r02r_sweep.txt 2>&1
}
run b1 HETM_TX_BLOCKS_PER_SM=1
run b2 HETM_TX_BLOCKS_PER_SM=2
run b1_amax HETM_TX_BLOCKS_PER_SM=1 HETM_APPLY_AMAX=1
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/r02r_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02r_tests.log
timeout 1500 ncu --set full --clock-control none -o /tmp/r02r_all python tools/ncu_all.py > gpurun_out/r02r_ncu_all.log 2>&1
python tools/summarize_ncu.py report /tmp/r02r_all.ncu-rep > gpurun_out/r02r_ncu_all_summary.txt 2>&1
du -sh gpurun_out
