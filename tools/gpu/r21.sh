mkdir -p gpurun_out/r21
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q > gpurun_out/r21/pytest_k.log 2>&1; tail -n 2 gpurun_out/r21/pytest_k.log
timeout 1200 python -m pytest tests/test_gpu_c5_sweep.py -x -q > gpurun_out/r21/pytest_sweep.log 2>&1; tail -n 2 gpurun_out/r21/pytest_sweep.log
timeout 1800 python tools/bench_c5.py --points all > gpurun_out/r21/c5_all.jsonl 2> gpurun_out/r21/c5_all.err; wc -l gpurun_out/r21/c5_all.jsonl; grep -v "^\s*$" gpurun_out/r21/c5_all.err | tail -n 3
