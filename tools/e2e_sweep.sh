# e2e round phase sweep (not product code): merge threads x zero-copy fraction
for t in 15 12; do for z in 0 0.15; do echo "threads=$t zc=$z"; HETM_MERGE_THREADS=$t HETM_ZC_FRACTION=$z python tools/e2e_probe.py 2>&1 | tail -3 | head -1; done; done
