mkdir -p gpurun_out/r12
timeout 1800 python -m pytest tests -m gpu -x -q --durations=15 > gpurun_out/r12/pytest_gpu.log 2>&1; tail -n 25 gpurun_out/r12/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r12/smoke.log 2>&1; tail -n 2 gpurun_out/r12/smoke.log
timeout 600 python bench.py > gpurun_out/r12/bench.json 2> gpurun_out/r12/bench.err; cat gpurun_out/r12/bench.json | cut -c1-400
