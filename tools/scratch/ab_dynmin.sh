#!/bin/bash
for m in 8388608 2097152 524288; do
  for mv in 0; do
  MPXA_DYN_MIN=$m SIZES=16384,65536,262144,1048576 timeout 300 python tools/tune_mid.py 2>&1 | head -1 | sed "s/^/min=$m /"
  MPXA_DYN_MIN=$m timeout 300 python tools/tune_a2av.py 2>&1 | tail -1 | sed "s/^/min=$m /"
  done
done
