# 2^24 stripes + AUTO 1/40: GPU suite, full bench (both arms), ncu of the bank kernel + apply
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/r02y_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02y_tests.log
timeout 900 python bench.py > gpurun_out/r02y_bench.json 2> gpurun_out/r02y_bench.err; echo "rc=$?" >> gpurun_out/r02y_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/r02y_bench_ref.json 2> gpurun_out/r02y_bench_ref.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"bank_batch_kernel|apply_xchg" -c 4 -o /tmp/r02y python tools/ncu_all.py > gpurun_out/r02y_ncu.log 2>&1
python tools/summarize_ncu.py report /tmp/r02y.ncu-rep > gpurun_out/r02y_ncu_summary.txt 2>&1
