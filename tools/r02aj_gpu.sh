# single counters memset: GPU suite, then the round's final bench line (both arms)
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/r02aj_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02aj_tests.log
timeout 900 python bench.py > gpurun_out/r02aj_bench.json 2> gpurun_out/r02aj_bench.err; echo "rc=$?" >> gpurun_out/r02aj_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/r02aj_bench_ref.json 2> gpurun_out/r02aj_bench_ref.err
