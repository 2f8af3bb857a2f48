timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
for l in 17 20 22 24; do timeout 120 python tools/probe_r02.py val $l; done
timeout 300 python bench.py --cpu-seconds 2 2>/dev/null
