# stripe bank kernel phase knockouts (EXPERIMENTS=1 build made on the box; some knockouts are incorrect)
mkdir -p gpurun_out
make -C paper_1905_00661_b200/csrc clean all EXPERIMENTS=1 > gpurun_out/r02t_build.log 2>&1
run() {  # tag, env...
  tag=$1; shift
  env "$@" timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --live-rounds 0 --no-configs --no-cfg5 --e2e-steps 2 > /tmp/b.json 2>/dev/null
  python -c "
import json,sys;l=json.loads(open('/tmp/b.json').readline());b=l['step_breakdown_ms']
print('$tag', 'step %.4f batch %.4f va %.4f merge %.4f aborts %d' % (b['step'],b['batch'],b['validate_apply'],b['merge_stage'],l['batch']['aborts_last']))" >> gpurun_out/r02t_knockouts.txt 2>&1
}
run product
run no_bitmaps HETM_STRIPE_KO=4
run no_ticket HETM_STRIPE_KO=1024
run no_validate HETM_STRIPE_KO=512
run no_fence HETM_STRIPE_KO=16384
run none_of_them HETM_STRIPE_KO=99
run product_again
