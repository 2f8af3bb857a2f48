# three default bench lines back to back (run-to-run spread of the final code)
mkdir -p gpurun_out
for i in 1 2 3; do timeout 900 python bench.py > gpurun_out/r02ap_bench_$i.json 2> gpurun_out/r02ap_bench_$i.err; done
