#!/bin/bash
# ncu --set full captures of the session-3 kernels (each command first run plain):
#   eager (LL) small alltoall on 4 emulated GPUs, variable-piece neighbor exchange,
#   resolved-move small alltoall on one GPU, partitioned Pready.
set -u
mkdir -p gpurun_out
run() {  # name, kernel regex, skip, command...
  local name=$1 rx=$2 skip=$3; shift 3
  timeout 300 "$@" > gpurun_out/plain_$name.log 2>&1 || { echo "$name plain failed"; return; }
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$rx -s $skip -c 1 \
      -o gpurun_out/prof_$name -f "$@" > gpurun_out/ncu_$name.log 2>&1; echo "$name ncu rc=$?"
}
run ll_a2a_1KiB_emu4 small_kernel 3 env EMU=4 B=1024 ALGO=pairwise python tools/scratch/one_a2a.py
run var_neighbor_random small_kernel 3 python tools/scratch/one_nb.py
run loc_bruck_16B small_kernel 3 env B=16 ALGO=bruck python tools/scratch/one_a2a.py
run part_pready_4KiB part_pready 3 python tools/scratch/tune_part.py
