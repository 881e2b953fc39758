#!/bin/bash
# A/B of libmpxa builds: default vs paper_2309_07337_b200/variants/*.so (VARIANTS="a b")
for v in default ${VARIANTS}; do
  if [ $v = default ]; then unset MPXA_LIB; else export MPXA_LIB=$PWD/paper_2309_07337_b200/variants/libmpxa_$v.so; fi
  echo "== $v"
  timeout 300 python tools/tune_copy.py 2>&1 | tail -1
  SIZES=65536,262144,1048576,4194304 timeout 300 python tools/tune_mid.py 2>&1 | head -1
  timeout 300 python tools/tune_a2av.py 2>&1 | tail -1
done
