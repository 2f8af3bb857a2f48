# robustness of the final code: full GPU suite under memcheck, racecheck of the shared-memory kernels, 2x soak
mkdir -p gpurun_out
timeout 3000 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests -m gpu -q -p no:cacheprovider -x --deselect tests/test_bench_contract.py > gpurun_out/r02ao_memcheck_full.log 2>&1; echo "rc=$?" >> gpurun_out/r02ao_memcheck_full.log
timeout 1200 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_bank_schedule.py tests/test_merge_stage.py -m gpu -q -p no:cacheprovider -x > gpurun_out/r02ao_racecheck.log 2>&1; echo "rc=$?" >> gpurun_out/r02ao_racecheck.log
for i in 1 2; do timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02ao_soak_$i.log 2>&1; echo "rc=$?" >> gpurun_out/r02ao_soak_$i.log; done
