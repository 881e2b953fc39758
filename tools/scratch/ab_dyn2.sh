#!/bin/bash
# dynamic mode: pieces per CTA x TMA ring config
for big in auto 0 1; do
 for pc in 8 16 32 64; do
  if [ $big = auto ]; then unset MPXA_TMA_BIG; else export MPXA_TMA_BIG=$big; fi
  MPXA_DYN_PIECES=$pc SIZES=1048576,4194304,16777216 timeout 300 python tools/tune_mid.py 2>&1 | head -1 | sed "s/^/big=$big pieces=$pc /"
 done
done
unset MPXA_TMA_BIG
for pc in 8 16 32 64; do MPXA_DYN_PIECES=$pc timeout 300 python tools/tune_copy.py 2>&1 | tail -1 | cut -c1-200 | sed "s/^/pieces=$pc /"; done
