#!/bin/bash
# One gpurun call: bench (plain), then the ncu launch list and one full capture of the
# top kernel on the SAME short command (run plain first, per B200_PROFILING.md).
set -u
mkdir -p gpurun_out
TAG=${TAG:-r01}
SHORT="python bench.py --no-sweep --no-e2e --no-cpu --steps 5 --warmup 3"
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/clocks_start_${TAG}.csv 2>&1
timeout 900 python bench.py ${BENCH_ARGS:-} --write-selector gpurun_out/selector_${TAG}.txt > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err; echo "bench rc=$?"
tail -c 3000 gpurun_out/bench_${TAG}.json
if [ "${NCU:-1}" = "1" ]; then
  timeout 300 $SHORT > gpurun_out/short_${TAG}.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
      --log-file gpurun_out/launches_${TAG}.csv $SHORT > gpurun_out/ncu_launch_${TAG}.log 2>&1; echo "ncu launches rc=$?"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:mpxa_exec -s 3 -c 1 \
      -o gpurun_out/prof_${TAG} -f $SHORT > gpurun_out/ncu_full_${TAG}.log 2>&1; echo "ncu full rc=$?"
fi
