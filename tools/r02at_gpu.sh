mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02at_gpu.txt 2>&1
timeout 900 python bench.py > gpurun_out/r02at_bench_n1.json 2> gpurun_out/r02at_bench_n1.err
timeout 600 python bench.py --impl reference > gpurun_out/r02at_bench_reference_n1.json 2> gpurun_out/r02at_bench_reference_n1.err
timeout 300 python tools/cache_sched_timeline.py > gpurun_out/r02at_cache_timeline.txt 2>&1
