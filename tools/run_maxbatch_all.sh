#!/bin/bash
# Max-batch sweep of the BASELINE models at 8 and 4 stages under a 40 GiB
# per-GPU cap (Table 2 of the paper); one JSON result per (model, stages).
# usage: tools/run_maxbatch_all.sh "gpt2-xl:8:64 t5-large:8:512" [outdir]
out=${2:-gpurun_out/maxbatch}
mkdir -p "$out"
for spec in $1; do
  IFS=: read model stages bmax <<< "$spec"
  timeout 3000 python tools/max_batch.py --model "$model" --stages "$stages" --b-max "$bmax" \
     --calibrate --out "$out/${model}_l${stages}.json" > "$out/${model}_l${stages}.log" 2>&1
  echo "$model l=$stages rc=$? $(tail -1 "$out/${model}_l${stages}.log" | cut -c1-600)"
done
