# HEAD measurement: full GPU suite, bench (both arms), launch list, ncu --set full of every product kernel
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02k_gpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/r02k_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02k_tests.log
timeout 900 python bench.py > gpurun_out/r02k_bench.json 2> gpurun_out/r02k_bench.err; echo "rc=$?" >> gpurun_out/r02k_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/r02k_bench_ref.json 2> gpurun_out/r02k_bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02k_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-preroll --live-rounds 0 --no-configs --no-cfg5 > gpurun_out/r02k_launches.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -o /tmp/r02k_all python tools/ncu_all.py > gpurun_out/r02k_ncu_all.log 2>&1
python tools/summarize_ncu.py report /tmp/r02k_all.ncu-rep > gpurun_out/r02k_ncu_all_summary.txt 2>&1
ncu -i /tmp/r02k_all.ncu-rep --page raw --csv 2>/dev/null | gzip -c > gpurun_out/r02k_ncu_all_raw.csv.gz
cp /tmp/r02k_all.ncu-rep gpurun_out/ 2>/dev/null
ls -la gpurun_out/ >> gpurun_out/r02k_ncu_all.log
