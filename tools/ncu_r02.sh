#!/bin/bash
# ncu --set full captures of the round-2 kernel paths (each command first run plain, one GPU):
#   tiny one-step (alltoall p=8, 16 B), tiny multi-step with owned flows (ring allgather 4 KiB),
#   tiny eager on 4 emulated GPUs (alltoall 16 B), the small kernel's 8-byte path (cfg4 mean
#   64 KiB), the dynamic executor at a mid size (allgather 4 MiB), the warp rings (cfg4 4 MiB).
set -u
mkdir -p gpurun_out
run() {  # name, kernel regex, skip, env assignments...
  local name=$1 rx=$2 skip=$3; shift 3
  env "$@" timeout 300 python tools/one_launch.py > gpurun_out/plain_$name.log 2>&1 || { echo "$name plain failed"; return; }
  env "$@" timeout 600 ncu --set full --clock-control none --import-source on -k regex:$rx -s $skip -c 1 \
      -o gpurun_out/prof_$name -f python tools/one_launch.py > gpurun_out/ncu_$name.log 2>&1; echo "$name ncu rc=$?"
}
run tiny_a2a_16B tiny_kernel 3 OP=alltoall B=16
run tiny_ms_ring_ag_4KiB tiny_ms 3 OP=allgather ALGO=ring B=4096
run tiny_ll_a2a_16B_emu4 tiny_ll 3 OP=alltoall B=16 EMU=4
run small_a2av_cfg4_64KiB mpxa_ 3 OP=alltoallv B=65536
run dyn_ag_4MiB mpxa_exec 3 OP=allgather B=4194304
run wring_a2av_cfg4_4MiB mpxa_exec 3 OP=alltoallv B=4194304
