# ncu --set full of the stripe bank kernel and the exchange apply (source-level stalls)
mkdir -p gpurun_out
export HETM_TX_BLOCKS_PER_SM=2
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"bank_batch_kernel|apply_xchg" -c 4 -o /tmp/r02o python tools/ncu_all.py > gpurun_out/r02o_ncu.log 2>&1
python tools/summarize_ncu.py report /tmp/r02o.ncu-rep > gpurun_out/r02o_ncu_summary.txt 2>&1
ncu -i /tmp/r02o.ncu-rep --page source --csv --print-source sass -k regex:bank_batch 2>/dev/null | gzip -c > gpurun_out/r02o_bank_source_sass.csv.gz
ncu -i /tmp/r02o.ncu-rep --page source --csv -k regex:bank_batch 2>/dev/null | gzip -c > gpurun_out/r02o_bank_source_cuda.csv.gz
ncu -i /tmp/r02o.ncu-rep --page raw --csv 2>/dev/null | gzip -c > gpurun_out/r02o_raw.csv.gz
du -sh gpurun_out/*
