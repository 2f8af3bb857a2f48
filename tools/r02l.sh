timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
for ko in 0 64; do HETM_KNOCKOUT=$ko timeout 120 python tools/probe_r02.py bank; done
timeout 120 python tools/probe_r02.py val 20
timeout 900 python tools/cfg5_sweep.py --gs 2,4,8 --logs-mib 64,1024 2>&1 | cut -c1-300
timeout 300 python bench.py --cpu-seconds 2 > gpurun_out/r02l.json 2>/dev/null
