#!/bin/bash
# ncu --set full captures of the dynamic-mode paths on the current build (cfg4 warp rings at
# mean 4 MiB, allgather 4 MiB producer ring, alltoall 1 MiB blocks) -- each command run plain
# first, one GPU (tools/one_launch.py).
set -u
mkdir -p gpurun_out
run() {  # name, kernel regex, skip, env assignments...
  local name=$1 rx=$2 skip=$3; shift 3
  env "$@" timeout 300 python tools/one_launch.py > gpurun_out/plain_$name.log 2>&1 || { echo "$name plain failed"; return; }
  env "$@" timeout 600 ncu --set full --clock-control none --import-source on -k regex:$rx -s $skip -c 1 \
      -o gpurun_out/prof_$name -f python tools/one_launch.py > gpurun_out/ncu_$name.log 2>&1; echo "$name ncu rc=$?"
}
run wring_a2av_cfg4_4MiB_${TAG:-s22} mpxa_exec 3 OP=alltoallv B=4194304
