for f in 0 0.2 0.35 0.5; do HETM_ZC_FRACTION=$f timeout 300 python tools/e2e_probe.py | sed "s/^/zc=$f /"; done
timeout 300 python -m pytest tests -m gpu -x -q -k "merge or live or cache_rounds" 2>&1 | tail -2
