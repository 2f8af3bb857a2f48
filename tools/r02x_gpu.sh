mkdir -p gpurun_out
for b in 22 23 24; do HETM_STRIPE_BITS=$b timeout 600 python tools/stripe_skew_probe.py >> gpurun_out/r02x_skew.txt 2>&1; done
