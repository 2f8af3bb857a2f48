for ko in 0 1; do HETM_KNOCKOUT=$ko timeout 120 python tools/probe_r02.py bank; done
timeout 600 python -m pytest tests -m gpu -x -q -k "bank or cfg2 or rounds" 2>&1 | tail -2
