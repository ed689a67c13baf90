mkdir -p gpurun_out/r49
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r49/pytest_gpu.log 2>&1; tail -n 2 gpurun_out/r49/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r49/smoke.log 2>&1; tail -n 1 gpurun_out/r49/smoke.log
timeout 600 python bench.py > gpurun_out/r49/bench_c4.json 2> gpurun_out/r49/bench_c4.err; python3 -c "import json; d=json.loads(open('gpurun_out/r49/bench_c4.json').readline()); print(d['value'], d['ms_per_step'], d['clocks'], d['e2e']['value'], d['roofline']['frac'], d['roofline']['kernel_ms'])"
timeout 2400 python tools/bench_c5.py --points all > gpurun_out/r49/c5_all.jsonl 2> gpurun_out/r49/c5_all.err; wc -l gpurun_out/r49/c5_all.jsonl; grep -v "^\s*$" gpurun_out/r49/c5_all.err | tail -n 2
