for ko in 0 2048 0 2048; do HETM_KNOCKOUT=$ko timeout 120 python tools/probe_r02.py bank; done
HETM_KNOCKOUT=2048 timeout 600 python -m pytest tests -m gpu -x -q -k "bank or cfg2 or cfg3 or rounds or merge" 2>&1 | tail -3
HETM_KNOCKOUT=2048 timeout 300 python tools/zipf_probe.py 2>&1 | head -6
