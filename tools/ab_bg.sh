#!/bin/bash
# A/B of the fused kernel's batch-group size (EPHDC_F64_BG), same box
O=gpurun_out/${1:-abbg}; mkdir -p $O
for r in 1 2; do
  for bg in 8 16 29 4; do
    EPHDC_F64_BG=$bg timeout 600 python bench.py --config c4 --no-e2e --no-cpu > $O/c4_bg${bg}_r$r.json 2>$O/err_bg${bg}_r$r.txt
  done
done
