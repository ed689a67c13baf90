mkdir -p gpurun_out/r5
cp ablibs/libB.so paper_2511_00737_b200/libephdc.so
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -k "c5 or fwd_inv" > gpurun_out/r5/pytest_B.log 2>&1; tail -2 gpurun_out/r5/pytest_B.log
cp ablibs/libA.so paper_2511_00737_b200/libephdc.so
POINTS="13:fwd 12:fwd" tools/ab_c5.sh r5
