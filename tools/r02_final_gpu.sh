# final measurements of the round: bench N=1 (both arms), launch list, warm ncu of the step kernels
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > gpurun_out/final_gpu.txt 2>&1
timeout 900 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; echo "rc=$?" >> gpurun_out/final_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/final_bench_ref.json 2> gpurun_out/final_bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file gpurun_out/final_launches.csv python bench.py --steps 6 --warmup 5 --e2e-steps 1 --no-cpu-baseline --no-preroll --live-rounds 0 --no-configs --no-cfg5 > gpurun_out/final_launches.log 2>&1
timeout 900 ncu --set full --cache-control none --clock-control none -k regex:"bank_batch_kernel|apply_xchg|delta_|winner|clear_round" -s 10 -c 6 -o /tmp/final_warm python bench.py --steps 6 --warmup 5 --no-cpu-baseline --no-preroll --live-rounds 0 --no-configs --no-cfg5 --e2e-steps 1 > gpurun_out/final_ncu.log 2>&1
python tools/summarize_ncu.py report /tmp/final_warm.ncu-rep > gpurun_out/final_ncu_warm_summary.txt 2>&1
