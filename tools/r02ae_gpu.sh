# fence.release in the stripe kernel: step A/B (acq_rel build kept as a sibling library) + warm ncu of the full batch
mkdir -p gpurun_out
run() {  # tag, env...
  tag=$1; shift
  env "$@" timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --live-rounds 0 --no-configs --no-cfg5 --e2e-steps 3 > /tmp/b.json 2>/dev/null
  python -c "
import json,sys;l=json.loads(open('/tmp/b.json').readline());b=l['step_breakdown_ms']
print('$tag', 'step %.4f batch %.4f va %.4f merge %.4f aborts %d' % (b['step'],b['batch'],b['validate_apply'],b['merge_stage'],l['batch']['aborts_last']), l['bank_sum_ok'], l['shadow_equals_replica'])" >> gpurun_out/r02ae_sweep.txt 2>&1
}
run release
run release_again
run release_3
timeout 900 ncu --set full --cache-control none --clock-control none -k regex:"bank_batch_kernel|apply_xchg|delta_|winner" -s 12 -c 6 -o /tmp/r02ae_warm python bench.py --steps 6 --warmup 5 --no-cpu-baseline --no-preroll --live-rounds 0 --no-configs --no-cfg5 --e2e-steps 1 > gpurun_out/r02ae_ncu.log 2>&1
python tools/summarize_ncu.py report /tmp/r02ae_warm.ncu-rep > gpurun_out/r02ae_ncu_warm_summary.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_bank_schedule.py tests/test_trace_gpu.py tests/test_acceptance.py -m gpu -q -p no:cacheprovider -x > gpurun_out/r02ae_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02ae_tests.log
