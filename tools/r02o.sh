timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests -m gpu -x -q -k "spec or clear_round or validate_apply_matches or hot_words or merge_commit_one or cache_batch_replays and 64 or route_log" 2>&1 | tail -15 > gpurun_out/memcheck.log
timeout 600 /usr/local/cuda/bin/compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests -m gpu -x -q -k "route_log and 100003 or validate_apply_matches and 8" 2>&1 | tail -15 > gpurun_out/racecheck.log
timeout 300 python tools/e2e_probe.py > gpurun_out/e2e_probe.txt 2>&1
