# step timeline (CUPTI) + full bench line of HEAD
mkdir -p gpurun_out
timeout 300 python tools/bench_step_timeline.py > gpurun_out/r02q_step_timeline.txt 2>&1
timeout 900 python bench.py > gpurun_out/r02q_bench.json 2> gpurun_out/r02q_bench.err; echo "rc=$?" >> gpurun_out/r02q_bench.err
