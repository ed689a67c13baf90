mkdir -p gpurun_out/r7
timeout 1200 python -m pytest tests -m gpu -x -q --deselect tests/test_gpu_c5_sweep.py --deselect tests/test_gpu_fullsize.py > gpurun_out/r7/pytest_gpu.log 2>&1; tail -5 gpurun_out/r7/pytest_gpu.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r7/bench_c4.json 2> gpurun_out/r7/bench_c4.err; tail -c 3000 gpurun_out/r7/bench_c4.json
