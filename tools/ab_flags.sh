#!/bin/bash
# A/B of workspace launch-plan overrides (ephdc_plan via bench.py --plan) on the same box.
# usage: tools/ab_flags.sh <tag> "<plan> <plan> ..." [configs...]   e.g. "flags=0 flags=2 bg=8"
O=gpurun_out/$1; PL=$2; shift 2; CFGS=${@:-c4}; mkdir -p $O
for r in 1 2; do
  for p in $PL; do
    for c in $CFGS; do
      timeout 600 python bench.py --config $c --no-e2e --no-cpu --plan "$p" > $O/${c}_${p}_r$r.json 2>$O/err_${c}_${p}_r$r.txt
    done
  done
done
