# A/B: evict-first (st.global.cs) stores for the merge stage's records and devShadow refresh vs plain stores
mkdir -p gpurun_out
ARGS="--steps 20 --warmup 5 --no-cpu-baseline --live-rounds 0 --no-configs --no-cfg5 --e2e-steps 10"
for i in 1 2 3; do
  for v in base cs; do
    cp abvar/$v/libhetm_b200.so paper_1905_00661_b200/libhetm_b200.so
    timeout 300 python bench.py $ARGS 2>/dev/null | grep '^{' > gpurun_out/r02az_${v}_$i.json
  done
done
cp abvar/cs/libhetm_b200.so paper_1905_00661_b200/libhetm_b200.so
timeout 900 python -m pytest tests -m gpu -x -q -k "merge or delta or shadow or rollback or abort" > gpurun_out/r02az_cs_tests.log 2>&1
