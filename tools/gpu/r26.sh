mkdir -p gpurun_out/r26
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_sr.py -x -q > gpurun_out/r26/pytest_k.log 2>&1; tail -n 2 gpurun_out/r26/pytest_k.log
timeout 1500 python -m pytest tests/test_gpu_c5_sweep.py -x -q > gpurun_out/r26/pytest_sweep.log 2>&1; tail -n 2 gpurun_out/r26/pytest_sweep.log
for spec in "14 3 48 fwd 65536" "16 9 30 fwd 7281" "15 5 48 fwd 26214"; do
  set -- $spec
  for rep in 1 2 3; do echo -n "fwd $spec rep$rep: "; timeout 120 python tools/c5_point.py --lg $1 --L $2 --bits $3 --op $4 --batch $5 --reps 100 2>&1 | tail -n 1 | cut -c1-100; done
done
cp paper_2511_00737_b200/libephdc.so /tmp/lib_orig.so
cp ablibs/libI.so paper_2511_00737_b200/libephdc.so
for spec in "14 3 48 inv 65536" "16 9 30 inv 7281" "15 5 48 inv 26214"; do
  set -- $spec
  for rep in 1 2 3 4; do echo -n "invcl2g $spec rep$rep: "; timeout 120 python tools/c5_point.py --lg $1 --L $2 --bits $3 --op $4 --batch $5 --reps 100 2>&1 | tail -n 1 | cut -c1-100; done
done
timeout 300 python -m pytest tests/test_gpu_kernels.py -x -q -k "two_groups or prime_switch or fwd_inv" > gpurun_out/r26/pytest_invcl2g.log 2>&1; tail -n 2 gpurun_out/r26/pytest_invcl2g.log
cp /tmp/lib_orig.so paper_2511_00737_b200/libephdc.so
EXTRA="--points all" LIBS="A B" POINTS="13:9:48:8 14:9:48:8 12:16:30:8 13:5:30:8 16:3:48:8" bash tools/ab_c5libs.sh r26/ab | grep mac
