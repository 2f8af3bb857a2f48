# final check of HEAD: smoke + full GPU suite
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02as_smoke.txt 2>&1; echo "rc=$?" >> gpurun_out/r02as_smoke.txt
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02as_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02as_tests.log
