#!/bin/bash
O=gpurun_out/r64; mkdir -p $O
for mb in 0 15 8 4; do
  if [ $mb = 0 ]; then P=""; else P="--plan m_batches=$mb"; fi
  timeout 600 python bench.py --config c4 --no-cpu --no-e2e $P > $O/bench_c4_mb$mb.json 2> $O/bench_c4_mb$mb.err; echo "mb $mb rc=$?" >> $O/rc.txt
done
