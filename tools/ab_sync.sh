#!/bin/bash
# A/B of the fused kernel's synchronisation variants (EPHDC_F64_FLAGS bits 1-2), same box
O=gpurun_out/${1:-ab2}; mkdir -p $O
for r in 1 2; do
  for f in 0 2 4; do
    EPHDC_F64_FLAGS=$f timeout 600 python bench.py --config c4 --no-e2e --no-cpu > $O/c4_f${f}_r$r.json 2>$O/err_f${f}_r$r.txt
    EPHDC_F64_FLAGS=$f timeout 600 python bench.py --config c3 --no-e2e --no-cpu > $O/c3_f${f}_r$r.json 2>>$O/err_f${f}_r$r.txt
  done
done
