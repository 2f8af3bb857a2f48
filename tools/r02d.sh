timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
timeout 300 python bench.py --cpu-seconds 2 2>&1 | tail -3
timeout 300 python bench.py --no-cpu-baseline --chunk-merge --steps 5 2>&1 | tail -1 | python -c "import json,sys; print('chunk-merge e2e', json.loads(sys.stdin.read())['e2e'])"
