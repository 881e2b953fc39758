#!/bin/bash
# A/B: dynamic work queue on/off (device us per call in CUDA graphs)
for v in 0 1; do
  MPXA_NO_DYN=$v SIZES=65536,262144,1048576,4194304,16777216 timeout 300 python tools/tune_mid.py 2>&1 | head -1 | sed "s/^/nodyn=$v /"
  MPXA_NO_DYN=$v timeout 300 python tools/tune_copy.py 2>&1 | tail -1 | sed "s/^/nodyn=$v /"
done
