mkdir -p gpurun_out/r17
timeout 300 python -m pytest tests/test_gpu_kernels.py -x -q -k "two_groups" > gpurun_out/r17/pytest_2g.log 2>&1; tail -n 3 gpurun_out/r17/pytest_2g.log
timeout 600 python -m pytest tests/test_gpu_variants.py -x -q > gpurun_out/r17/pytest_var.log 2>&1; tail -n 3 gpurun_out/r17/pytest_var.log
if grep -q " passed" gpurun_out/r17/pytest_var.log && ! grep -q "failed\|error" gpurun_out/r17/pytest_var.log; then
  for r in 1 2; do
    timeout 600 python bench.py --no-cpu --no-e2e > gpurun_out/r17/bench_2g_r$r.json 2>/dev/null
    timeout 600 python bench.py --no-cpu --no-e2e --plan flags=32 > gpurun_out/r17/bench_1t_r$r.json 2>/dev/null
    timeout 600 python bench.py --config c3 --no-cpu --no-e2e --steps 20 > gpurun_out/r17/bench_c3_2g_r$r.json 2>/dev/null
    timeout 600 python bench.py --config c3 --no-cpu --no-e2e --steps 20 --plan flags=32 > gpurun_out/r17/bench_c3_1t_r$r.json 2>/dev/null
  done
  python3 -c "
import json,glob
for f in sorted(glob.glob('gpurun_out/r17/bench_*.json')):
    try: d=json.loads(open(f).readline()); print(f.split('/')[-1], d['value'], d['ms_per_step'], d['roofline']['kernel_ms'].get('ntt_mac'), d['clocks'].get('sm_mhz'), d['clocks'].get('reasons'))
    except Exception as e: print(f, 'ERR', e)
"
fi
if grep -q " passed" gpurun_out/r17/pytest_2g.log && ! grep -q "failed\|error" gpurun_out/r17/pytest_2g.log; then
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q > gpurun_out/r17/pytest_k.log 2>&1; tail -n 2 gpurun_out/r17/pytest_k.log
for r in 1 2; do
timeout 300 python tools/bench_c5.py --only 14:9:48:8,15:5:48:8,16:3:48:8 --max-batch-only > gpurun_out/r17/c5_new_r$r.jsonl 2>/dev/null
timeout 300 python tools/bench_c5.py --only 14:9:48:8,15:5:48:8,16:3:48:8 --max-batch-only --alt-teams > gpurun_out/r17/c5_alt_r$r.jsonl 2>/dev/null
done
python3 -c "
import json,glob
for f in sorted(glob.glob('gpurun_out/r17/c5_*.jsonl')):
    for l in open(f):
        r=json.loads(l)
        if 'ntt_fwd' in r: print(f.split('/')[-1], r['log2N'],r['L'],r['bits'],r['batch'],r['ntt_fwd']['frac_hbm'],r['ntt_inv']['frac_hbm'],r['clocks'].get('sm_mhz'), r['clocks'].get('reasons'))
"
fi
