set -x; mkdir -p gpurun_out/r3
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q > gpurun_out/r3/pytest_kernels.log 2>&1; tail -15 gpurun_out/r3/pytest_kernels.log
for op in fwd inv; do for lg in 12 13 14; do timeout 120 python tools/c5_point.py --lg $lg --L 9 --bits 48 --op $op --reps 5; done; done > gpurun_out/r3/c5.log 2>&1
cat gpurun_out/r3/c5.log
timeout 120 python tools/c5_point.py --lg 13 --L 9 --bits 48 --op fwd --batch 2048 --reps 1 && \
ncu --set full --clock-control none --import-source on -k regex:k_ntt_c5 -c 1 -o gpurun_out/r3/fwd13 python tools/c5_point.py --lg 13 --L 9 --bits 48 --op fwd --batch 2048 --reps 1 > gpurun_out/r3/ncu1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_ntt_c5 -c 1 -o gpurun_out/r3/inv13 python tools/c5_point.py --lg 13 --L 9 --bits 48 --op inv --batch 2048 --reps 1 > gpurun_out/r3/ncu2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_ntt_c5 -c 1 -o gpurun_out/r3/fwd14 python tools/c5_point.py --lg 14 --L 9 --bits 48 --op fwd --batch 1024 --reps 1 > gpurun_out/r3/ncu3.log 2>&1
tail -n 2 gpurun_out/r3/ncu*.log
