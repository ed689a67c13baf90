set -x; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
for op in fwd inv; do for lg in 13 14; do python tools/c5_point.py --lg $lg --L 9 --bits 48 --op $op --reps 5; done; done > gpurun_out/c5_base.log 2>&1
cat gpurun_out/c5_base.log
python tools/c5_point.py --lg 13 --L 9 --bits 48 --op fwd --batch 2048 --reps 1 && \
ncu --set full --clock-control none --import-source on -k regex:k_ntt_std -s 1 -c 1 -o gpurun_out/c5_fwd13 python tools/c5_point.py --lg 13 --L 9 --bits 48 --op fwd --batch 2048 --reps 1 > gpurun_out/ncu1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_ntt_std -s 1 -c 1 -o gpurun_out/c5_inv13 python tools/c5_point.py --lg 13 --L 9 --bits 48 --op inv --batch 2048 --reps 1 > gpurun_out/ncu2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_ntt_std -s 1 -c 1 -o gpurun_out/c5_fwd14 python tools/c5_point.py --lg 14 --L 9 --bits 48 --op fwd --batch 1024 --reps 1 > gpurun_out/ncu3.log 2>&1
tail -3 gpurun_out/ncu*.log
