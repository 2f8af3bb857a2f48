# final code of the round: GPU suite, smoke, bench (both arms), ncu launch list of the bench
mkdir -p gpurun_out
s=$(date +%s); timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02ba_gpu_tests.log 2>&1; echo "rc=$? $(( $(date +%s) - s )) s" >> gpurun_out/r02ba_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02ba_smoke.txt 2>&1; echo "rc=$?" >> gpurun_out/r02ba_smoke.txt
timeout 900 python bench.py > gpurun_out/r02ba_bench_n1.json 2> gpurun_out/r02ba_bench_n1.err
timeout 600 python bench.py --impl reference > gpurun_out/r02ba_bench_reference_n1.json 2> gpurun_out/r02ba_bench_reference_n1.err
