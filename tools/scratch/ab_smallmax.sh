#!/bin/bash
for mv in "1048576 16777216" "4194304 33554432" "4194304 67108864"; do
  set -- $mv
  MPXA_SMALL_MAX=$1 MPXA_SMALL_VOL=$2 SIZES=524288,1048576,2097152,4194304 timeout 300 python tools/tune_mid.py 2>&1 | head -1 | sed "s/^/max=$1 vol=$2 /"
done
