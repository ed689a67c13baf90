#!/bin/bash
# A/B(/C...) of builds of libephdc.so (ablibs/libA.so, ablibs/libB.so, ...) on the same box.
# usage: [LIBS="A B C"] tools/ab_libs.sh <tag> [configs...]
O=gpurun_out/${1:-ablib}; shift; CFGS=${@:-c4}; mkdir -p $O
for r in 1 2; do
  for v in ${LIBS:-A B}; do
    for c in $CFGS; do
      EPHDC_LIB=$PWD/ablibs/lib$v.so timeout 600 python bench.py --config $c --no-e2e --no-cpu > $O/${c}_${v}_r$r.json 2>$O/err_${c}_${v}_r$r.txt
    done
  done
done
