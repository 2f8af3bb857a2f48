for n in 20 22 24; do for b in 1 2; do for u in 2 4 8; do HETM_APPLY_UNROLL=$u HETM_APPLY_BLOCKS_PER_SM=$b timeout 120 python tools/probe_r02.py val $n | sed "s/^/bps=$b u=$u /" | cut -c1-110; done; done; done
timeout 600 python tools/cfg5_sweep.py --gs 8 --logs-mib 64,1024 2>&1 | cut -c1-700
