#!/bin/bash
mkdir -p gpurun_out/exp14
o=gpurun_out/exp14
for rep in 1 2; do for v in lnb lnr4 lnr5 lnr2c3; do timeout 300 python tools/ln_ab.py abso/$v.so >> $o/ln_ab.jsonl 2>&1; done; done; cat $o/ln_ab.jsonl
