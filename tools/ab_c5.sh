#!/bin/bash
# A/B(/C...) of libephdc.so builds (ablibs/libX.so) on the c5 points, same box.
# usage: [LIBS="A B"] [POINTS="13:fwd 12:fwd"] tools/ab_c5.sh <tag>
O=gpurun_out/${1:-abc5}; mkdir -p $O
LIB=paper_2511_00737_b200/libephdc.so
cp $LIB $O/libephdc.orig.so
for r in 1 2; do
  for v in ${LIBS:-A B}; do
    cp ablibs/lib$v.so $LIB
    for pt in ${POINTS:-13:fwd 12:fwd 14:fwd}; do
      lg=${pt%%:*}; op=${pt##*:}
      echo "$v r$r $(timeout 120 python tools/c5_point.py --lg $lg --L 9 --bits 48 --op $op --reps 5)" >> $O/ab.txt
    done
  done
done
cp $O/libephdc.orig.so $LIB
cat $O/ab.txt
