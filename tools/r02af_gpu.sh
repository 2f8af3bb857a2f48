# 32-bit stripe words (2^24 = 64 MiB): step, skew/AUTO signal, warm ncu, GPU suite
mkdir -p gpurun_out
run() {  # tag, env...
  tag=$1; shift
  env "$@" timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --live-rounds 0 --no-configs --no-cfg5 --e2e-steps 3 > /tmp/b.json 2>/dev/null
  python -c "
import json,sys;l=json.loads(open('/tmp/b.json').readline());b=l['step_breakdown_ms']
print('$tag', 'step %.4f batch %.4f va %.4f merge %.4f aborts %d' % (b['step'],b['batch'],b['validate_apply'],b['merge_stage'],l['batch']['aborts_last']), l['bank_sum_ok'], l['shadow_equals_replica'])" >> gpurun_out/r02af_sweep.txt 2>&1
}
run s32_b24
run s32_b25 HETM_STRIPE_BITS=25
run s32_b24_again
timeout 600 python tools/stripe_skew_probe.py > gpurun_out/r02af_skew.txt 2>&1
timeout 900 ncu --set full --cache-control none --clock-control none -k regex:"bank_batch_kernel" -s 6 -c 2 -o /tmp/r02af_warm python bench.py --steps 6 --warmup 5 --no-cpu-baseline --no-preroll --live-rounds 0 --no-configs --no-cfg5 --e2e-steps 1 > gpurun_out/r02af_ncu.log 2>&1
python tools/summarize_ncu.py report /tmp/r02af_warm.ncu-rep > gpurun_out/r02af_ncu_warm_summary.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/r02af_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02af_tests.log
