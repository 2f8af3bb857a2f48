# host merge-scatter order probe (box CPU) + HEAD bench (both arms) + bench launch list
mkdir -p gpurun_out
./build/host_order_probe > gpurun_out/r02w_host_order_probe.txt 2>&1
timeout 900 python bench.py > gpurun_out/r02w_bench.json 2> gpurun_out/r02w_bench.err; echo "rc=$?" >> gpurun_out/r02w_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/r02w_bench_ref.json 2> gpurun_out/r02w_bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/r02w_launches.csv python bench.py --steps 6 --warmup 3 --e2e-steps 1 --no-cpu-baseline --no-preroll --live-rounds 0 --no-configs --no-cfg5 > gpurun_out/r02w_launches.log 2>&1
