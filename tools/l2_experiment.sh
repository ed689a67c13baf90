#!/bin/bash
# DRAM traffic / L2 reuse of the fused kernel under grid-order knobs (ncu metrics only).
O=gpurun_out/l2exp; mkdir -p $O
CMD="python bench.py --config c4 --steps 1 --warmup 3 --no-e2e --no-cpu"
timeout 600 $CMD > $O/plain.log 2>&1 || exit 1
for v in "0 8" "1 8" "0 1" "0 4" "0 16"; do
  set -- $v
  EPHDC_F64_FLAGS=$1 EPHDC_F64_BG=$2 timeout 900 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum --clock-control none -k regex:k_ntt_mac_f64 -s 3 -c 1 --csv $CMD > $O/flags$1_bg$2.csv 2> $O/flags$1_bg$2.err
done
