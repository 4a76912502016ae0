#!/bin/bash
# Max-batch sweep of the BASELINE models under a 40 GiB per-GPU cap (Table 2
# of the paper); one JSON result per spec.
# usage: tools/run_maxbatch_all.sh "gpt2-xl:8:64 t5-large:8:512[:strategies[:b_start]]" [outdir]
out=${2:-gpurun_out/maxbatch}
mkdir -p "$out"
for spec in $1; do
  IFS=: read model stages bmax strats bstart <<< "$spec"
  strats=${strats:-even_compute,even_compute_memopt,dawnpiper}
  tag=${model}_l${stages}${bstart:+_from$bstart}
  timeout 3000 python tools/max_batch.py --model "$model" --stages "$stages" --b-max "$bmax" \
     --strategies "$strats" --b-start "${bstart:-1}" \
     --calibrate --out "$out/$tag.json" > "$out/$tag.log" 2>&1
  echo "$model l=$stages rc=$? $(tail -1 "$out/$tag.log" | cut -c1-600)"
done
# timing-only specs: TIME="model:stages:STRAT:B,STRAT:B ..." tools/run_maxbatch_all.sh ""
for spec in $TIME; do
  IFS=: read model stages rest <<< "$spec"
  tag=${model}_l${stages}_timing
  timeout 3000 python tools/max_batch.py --model "$model" --stages "$stages" --calibrate \
     --time-at "$rest" --out "$out/$tag.json" > "$out/$tag.log" 2>&1
  echo "$model l=$stages timing rc=$? $(grep at_max "$out/$tag.log" | cut -c1-300)"
done
