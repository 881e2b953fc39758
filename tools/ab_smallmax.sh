#!/bin/bash
SIZES=8192,65536,262144,524288,1048576,2097152 timeout 300 python tools/tune_mid.py 2>&1 | head -1
timeout 300 python tools/tune_a2av.py 2>&1 | tail -1
timeout 300 python tools/tune_copy.py 2>&1 | tail -1
