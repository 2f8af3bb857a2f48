set -x
for ko in 0 16 32 64; do HETM_KNOCKOUT=$ko timeout 120 python tools/probe_r02.py bank; done
for w in 16 17 18 19 20 24; do HETM_VAL_WINDOW_LOG2=$w timeout 120 python tools/probe_r02.py val 20; done
for w in 17 18 24; do HETM_VAL_WINDOW_LOG2=$w timeout 120 python tools/probe_r02.py val 22; done
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
