mkdir -p gpurun_out/r45
for lg in 13 14; do for op in fwd inv; do
timeout 300 python tools/c5_point.py --lg $lg --L 9 --bits 30 --op $op --u32 --reps 3 > gpurun_out/r45/pt${lg}_$op.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_ntt32_c5 -s 2 -c 1 -o gpurun_out/r45/ncu_u32_${op}${lg} python tools/c5_point.py --lg $lg --L 9 --bits 30 --op $op --u32 --reps 3 > gpurun_out/r45/ncu_${op}${lg}.log 2>&1; tail -n 1 gpurun_out/r45/ncu_${op}${lg}.log
done; done
