./build/tlb_probe2 > gpurun_out/r02g_tlb_probe2.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/r02g_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02g_tests.log
timeout 1500 ncu --set full --clock-control none -o /tmp/r02g_all python tools/ncu_all.py > gpurun_out/r02g_ncu_all.log 2>&1
ncu -i /tmp/r02g_all.ncu-rep --page raw --csv > /tmp/r02g_raw.csv 2>/dev/null
python tools/summarize_ncu.py report /tmp/r02g_all.ncu-rep > gpurun_out/r02g_ncu_all_summary.txt 2>&1
gzip -c /tmp/r02g_raw.csv > gpurun_out/r02g_ncu_all_raw.csv.gz
ls -la gpurun_out/ >> gpurun_out/r02g_ncu_all.log
