#!/bin/bash
# A/B of EPHDC_F64_FLAGS values on the same box. usage: tools/ab_flags.sh <tag> "<flags...>" [configs...]
O=gpurun_out/$1; FL=$2; shift 2; CFGS=${@:-c4}; mkdir -p $O
for r in 1 2; do
  for f in $FL; do
    for c in $CFGS; do
      EPHDC_F64_FLAGS=$f timeout 600 python bench.py --config $c --no-e2e --no-cpu > $O/${c}_f${f}_r$r.json 2>$O/err_${c}_f${f}_r$r.txt
    done
  done
done
