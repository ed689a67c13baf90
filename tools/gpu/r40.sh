mkdir -p gpurun_out/r40
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/r40/smi.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r40/pytest_gpu.log 2>&1; tail -n 2 gpurun_out/r40/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r40/smoke.log 2>&1; tail -n 1 gpurun_out/r40/smoke.log
timeout 600 python bench.py > gpurun_out/r40/bench_c4.json 2> gpurun_out/r40/bench_c4.err; python3 -c "import json; d=json.loads(open('gpurun_out/r40/bench_c4.json').readline()); print(d['value'], d['ms_per_step'], d['clocks'], d['e2e']['value'], d['roofline']['frac'])"
