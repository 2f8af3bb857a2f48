# final-code check: GPU suite, smoke, bench (both arms)
mkdir -p gpurun_out
s=$(date +%s); timeout 1500 python -m pytest tests -m gpu -x -q --durations=8 > gpurun_out/r02ax_gpu_tests.log 2>&1; echo "rc=$? $(( $(date +%s) - s )) s" >> gpurun_out/r02ax_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02ax_smoke.txt 2>&1; echo "rc=$?" >> gpurun_out/r02ax_smoke.txt
timeout 900 python bench.py > gpurun_out/r02ax_bench_n1.json 2> gpurun_out/r02ax_bench_n1.err
timeout 600 python bench.py --impl reference > gpurun_out/r02ax_bench_reference_n1.json 2> gpurun_out/r02ax_bench_reference_n1.err
