O=gpurun_out/r62; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $O/smi.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; tail -n 2 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -n 1 $O/smoke.log
timeout 600 python bench.py > $O/bench_c4.json 2> $O/bench_c4.err; python3 -c "import json; d=json.loads(open('$O/bench_c4.json').readline()); print(d['value'], d['ms_per_step'], d['clocks'], d['e2e']['value'], d['roofline']['frac'], d['roofline']['kernel_ms'])"
for c in c3 c2 c1q3; do timeout 600 python bench.py --config $c > $O/bench_$c.json 2> $O/bench_$c.err; python3 -c "import json; d=json.loads(open('$O/bench_$c.json').readline()); print('$c', d['value'], d['e2e']['value'], d['clocks']['sm_mhz'], d['roofline']['frac'])"; done
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu"
timeout 600 $CMD > $O/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv $CMD > $O/ncu_launch.log 2>&1; echo "launch rc=$?"
