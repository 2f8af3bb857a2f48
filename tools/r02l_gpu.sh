# stripe/apply probe + HEAD bench (both arms) + bench launch list
mkdir -p gpurun_out
./build/stripe_probe > gpurun_out/r02l_stripe_probe.txt 2>&1
timeout 900 python bench.py > gpurun_out/r02l_bench.json 2> gpurun_out/r02l_bench.err; echo "rc=$?" >> gpurun_out/r02l_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/r02l_bench_ref.json 2> gpurun_out/r02l_bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02l_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-preroll --live-rounds 0 --no-configs --no-cfg5 > gpurun_out/r02l_launches.log 2>&1
du -sh gpurun_out
