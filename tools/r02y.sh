for cfg in "0 1" "4096 2" "4096 1" "0 2"; do set -- $cfg; HETM_KNOCKOUT=$1 HETM_TX_BLOCKS_PER_SM=$2 timeout 120 python tools/probe_r02.py bank | sed "s/^/bps=$2 /"; done
HETM_KNOCKOUT=4096 HETM_TX_BLOCKS_PER_SM=2 timeout 300 python -m pytest tests -m gpu -x -q -k "bank_batch_replays or cfg2" 2>&1 | tail -1
