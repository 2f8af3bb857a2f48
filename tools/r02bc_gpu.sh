# catch the intermittent 2-ranks-on-one-GPU hang and dump every rank's Python stack (SIGABRT + faulthandler)
mkdir -p gpurun_out
export PYTHONFAULTHANDLER=1 HETM_BENCH_BACKEND=gloo HETM_BENCH_ONE_GPU=1
desc() { for c in $(ps -o pid= --ppid $1); do echo $c; desc $c; done; }
for i in $(seq 1 12); do
  python bench.py --steps 3 --warmup 3 --gpus 2 --no-cpu-baseline --no-configs --live-rounds 0 --e2e-steps 3 --cfg5-reps 1 > gpurun_out/r02bc_run$i.out 2> gpurun_out/r02bc_run$i.err &
  P=$!
  for t in $(seq 1 60); do sleep 1; kill -0 $P 2>/dev/null || break; done
  if kill -0 $P 2>/dev/null; then
    echo "run$i HUNG" >> gpurun_out/r02bc_runs.txt
    ps -o pid,ppid,stat,wchan:32,cmd --forest -g $(ps -o sid= -p $P) >> gpurun_out/r02bc_runs.txt 2>&1
    for c in $(desc $P); do cat /proc/$c/cmdline | tr '\0' ' ' >> gpurun_out/r02bc_runs.txt; echo " [$c]" >> gpurun_out/r02bc_runs.txt; done
    for c in $(desc $P); do kill -ABRT $c; done
    sleep 5
    for c in $(desc $P) $P; do kill -9 $c; done
    break
  else
    wait $P; echo "run$i rc=$?" >> gpurun_out/r02bc_runs.txt
  fi
done
