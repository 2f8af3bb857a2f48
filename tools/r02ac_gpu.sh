# bits-24 variants of the step, warm ncu of the bank kernel + apply inside bench.py, memcheck of the new kernels
mkdir -p gpurun_out
run() {  # tag, env...
  tag=$1; shift
  env "$@" timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --live-rounds 0 --no-configs --no-cfg5 --e2e-steps 3 > /tmp/b.json 2>/dev/null
  python -c "
import json,sys;l=json.loads(open('/tmp/b.json').readline());b=l['step_breakdown_ms']
print('$tag', 'step %.4f batch %.4f va %.4f merge %.4f aborts %d' % (b['step'],b['batch'],b['validate_apply'],b['merge_stage'],l['batch']['aborts_last']), l['bank_sum_ok'], l['shadow_equals_replica'])" >> gpurun_out/r02ac_sweep.txt 2>&1
}
run product
run twopl HETM_STRIPE_2PL=1
run b2 HETM_TX_BLOCKS_PER_SM=2
run bits22 HETM_STRIPE_BITS=22
run apply_b2 HETM_APPLY_BLOCKS_PER_SM=2
run apply_b2_u2 HETM_APPLY_BLOCKS_PER_SM=2 HETM_APPLY_UNROLL=2
run apply_b1_u8 HETM_APPLY_UNROLL=8
run apply_b4_u2 HETM_APPLY_BLOCKS_PER_SM=4 HETM_APPLY_UNROLL=2
run product_again
# warm capture: no cache flush between replays, launches of the timed loop (skip init + warm-up)
timeout 900 ncu --set full --cache-control none --clock-control none -k regex:"bank_batch_kernel|apply_xchg" -s 20 -c 4 -o /tmp/r02ac_warm python bench.py --steps 6 --warmup 3 --no-cpu-baseline --no-preroll --live-rounds 0 --no-configs --no-cfg5 --e2e-steps 1 > gpurun_out/r02ac_ncu.log 2>&1
python tools/summarize_ncu.py report /tmp/r02ac_warm.ncu-rep > gpurun_out/r02ac_ncu_warm_summary.txt 2>&1
timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_parity.py tests/test_bank_schedule.py -m gpu -q -p no:cacheprovider -x -k "bank or validate or auto" > gpurun_out/r02ac_memcheck.log 2>&1; echo "rc=$?" >> gpurun_out/r02ac_memcheck.log
