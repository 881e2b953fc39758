#!/bin/bash
# TMA pipeline variants + CTA grid overrides (one gpurun call)
out=gpurun_out/tune_${TAG:-x}.jsonl; : > $out
COPY_REF=1 timeout 300 python tools/tune_copy.py >> $out 2>&1
for v in paper_2309_07337_b200/variants/*.so; do MPXA_LIB=$v timeout 300 python tools/tune_copy.py >> $out 2>&1; done
for ns in 148 444 592; do MPXA_NS=$ns timeout 300 python tools/tune_copy.py >> $out 2>&1; done
cat $out
