#!/bin/bash
# ncu --set full of selected kernels of the c4 bench step (after a plain run exits 0).
# usage: tools/gpu_ncu_kernels.sh <tag> <kernel-regex> <count> [config]
TAG=$1; KRE=$2; CNT=${3:-2}; CFG=${4:-c4}
O=gpurun_out/$TAG; mkdir -p $O
CMD="python bench.py --config $CFG --steps 1 --warmup 3 --no-e2e --no-cpu"
timeout 600 $CMD > $O/plain.log 2>&1 && echo "plain rc=0" >> $O/rc.txt && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"$KRE" -s ${SKIP:-2} -c $CNT -o $O/prof $CMD > $O/ncu_full.log 2>&1; echo "ncu rc=$?" >> $O/rc.txt
