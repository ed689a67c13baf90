#!/bin/bash
# dram bytes / L2 hit rate / duration of the fused kernel for library builds A and B
# (ablibs/libA.so, ablibs/libB.so: each is copied over the in-tree libephdc.so, as in
# tools/ab_libs.sh -- the binding loads only that path and reads no environment).
O=gpurun_out/${1:-ncuq}; mkdir -p $O
LIB=paper_2511_00737_b200/libephdc.so
cp $LIB $O/lib_orig.so
CMD="python bench.py --config c4 --steps 1 --warmup 3 --no-e2e --no-cpu"
for v in A B; do
  cp ablibs/lib$v.so $LIB
  timeout 600 $CMD > $O/plain_$v.log 2>&1 || continue
  timeout 900 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,lts__throughput.avg.pct_of_peak_sustained_elapsed,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:k_ntt_mac_f64 -s 3 -c 1 --csv $CMD > $O/ncu_$v.csv 2> $O/ncu_$v.err
done
cp $O/lib_orig.so $LIB; rm -f $O/lib_orig.so
