# dynamic-queue piece size (MPXA_DYN_PIECES) on single-GPU allgather / alltoall / cfg4 (p = 8)
mkdir -p gpurun_out
K=";MPXA_DYN_PIECES=1;MPXA_DYN_PIECES=2;MPXA_DYN_PIECES=3;MPXA_DYN_PIECES=4;MPXA_DYN_PIECES=8;MPXA_NO_SMALL=1;MPXA_NO_SMALL=1,MPXA_DYN_PIECES=2;MPXA_TMA_BIG=1,MPXA_DYN_PIECES=2"
KNOBS="$K" SIZES_MIB=2,4,8,16,64 timeout 600 python tools/ag_tail.py > gpurun_out/dyn_pieces_ag.txt 2>&1
P=8 KNOBS="$K" SIZES_KIB=1024,4096,16384 timeout 600 python tools/a2a_knobs.py > gpurun_out/dyn_pieces_a2a.txt 2>&1
VARIANTS='{"default": {}, "dp2": {"MPXA_DYN_PIECES": "2"}, "dp4": {"MPXA_DYN_PIECES": "4"}, "dp8": {"MPXA_DYN_PIECES": "8"}}' MEANS=1,4,8 ELEMS=8 timeout 600 python tools/cfg4_knobs.py > gpurun_out/dyn_pieces_cfg4.txt 2>&1
cat gpurun_out/dyn_pieces_*.txt
