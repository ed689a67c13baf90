mkdir -p gpurun_out/r6
for v in B C; do cp ablibs/lib$v.so paper_2511_00737_b200/libephdc.so
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -k "c5 or fwd_inv" > gpurun_out/r6/pytest_$v.log 2>&1; tail -1 gpurun_out/r6/pytest_$v.log; done
cp ablibs/libA.so paper_2511_00737_b200/libephdc.so
LIBS="A B C" POINTS="13:fwd 12:fwd 13:inv 12:inv" tools/ab_c5.sh r6
