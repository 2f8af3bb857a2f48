# stripe-lock bank kernel: occupancy variants of the bench step, then the GPU suite
mkdir -p gpurun_out
for b in 1 2 4; do
  HETM_TX_BLOCKS_PER_SM=$b timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --live-rounds 0 --no-configs --no-cfg5 > gpurun_out/r02m_bench_b$b.json 2> gpurun_out/r02m_bench_b$b.err
done
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/r02m_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02m_tests.log
du -sh gpurun_out
