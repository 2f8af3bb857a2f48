# smoke + memcheck of the kernels changed this round (32-bit stripes, adaptive apply, AUTO retry feedback, merge stage)
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02ak_smoke.txt 2>&1; echo "rc=$?" >> gpurun_out/r02ak_smoke.txt
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_parity.py tests/test_bank_schedule.py tests/test_merge_stage.py tests/test_merge_prepare.py -m gpu -q -p no:cacheprovider -x > gpurun_out/r02ak_memcheck.log 2>&1; echo "rc=$?" >> gpurun_out/r02ak_memcheck.log
timeout 900 compute-sanitizer --tool synccheck python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -x -k "bank or validate" > gpurun_out/r02ak_synccheck.log 2>&1; echo "rc=$?" >> gpurun_out/r02ak_synccheck.log
