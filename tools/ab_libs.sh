#!/bin/bash
# A/B(/C...) of builds of libephdc.so (ablibs/libA.so, ablibs/libB.so, ...) on the same box:
# each build is copied over the in-tree library (a scratch copy on the GPU box) before its run.
# usage: [LIBS="A B C"] tools/ab_libs.sh <tag> [configs...]
O=gpurun_out/${1:-ablib}; shift; CFGS=${@:-c4}; mkdir -p $O
LIB=paper_2511_00737_b200/libephdc.so
cp $LIB $O/libephdc.orig.so
for r in 1 2; do
  for v in ${LIBS:-A B}; do
    cp ablibs/lib$v.so $LIB
    for c in $CFGS; do
      timeout 600 python bench.py --config $c --no-e2e --no-cpu > $O/${c}_${v}_r$r.json 2>$O/err_${c}_${v}_r$r.txt
    done
  done
done
cp $O/libephdc.orig.so $LIB
