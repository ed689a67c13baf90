mkdir -p gpurun_out/r9
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_find_dmax.py -x -q > gpurun_out/r9/pytest_k.log 2>&1; tail -15 gpurun_out/r9/pytest_k.log
timeout 900 python -m pytest tests/test_gpu_c5_sweep.py -x -q -k "N16384 or N32768 or N65536" > gpurun_out/r9/pytest_sweep.log 2>&1; tail -5 gpurun_out/r9/pytest_sweep.log
timeout 600 python tools/bench_c5.py --points quick --max-batch-only > gpurun_out/r9/c5_quick.jsonl 2> gpurun_out/r9/c5_quick.err; cat gpurun_out/r9/c5_quick.jsonl | cut -c1-400
