for b in 0 1 2 3 4; do HETM_APPLY_BLOCKS_PER_SM=$b timeout 120 python tools/probe_r02.py val 20 | sed "s/^/bps=$b /"; done
for b in 0 2 4; do HETM_APPLY_BLOCKS_PER_SM=$b timeout 120 python tools/probe_r02.py val 22 | sed "s/^/bps=$b /"; done
timeout 600 python tools/cfg5_sweep.py --gs 2,8 --logs-mib 64,1024 2>&1 | cut -c1-400
