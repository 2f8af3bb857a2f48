for ko in 0 512 1024 1536 4 64; do HETM_KNOCKOUT=$ko timeout 120 python tools/probe_r02.py bank; done
for b in 1 2 3 4; do HETM_TX_BLOCKS_PER_SM=$b timeout 120 python tools/probe_r02.py bank | sed "s/^/bps=$b /"; done
for b in 1 2 4; do HETM_KNOCKOUT=64 HETM_TX_BLOCKS_PER_SM=$b timeout 120 python tools/probe_r02.py bank | sed "s/^/bps=$b /"; done
