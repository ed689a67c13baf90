mkdir -p gpurun_out/r16
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q > gpurun_out/r16/pytest_k.log 2>&1; tail -n 2 gpurun_out/r16/pytest_k.log
timeout 900 python -m pytest tests/test_gpu_c5_sweep.py -x -q -k "N8192 or N16384" > gpurun_out/r16/pytest_sweep.log 2>&1; tail -n 2 gpurun_out/r16/pytest_sweep.log
for r in 1 2; do
timeout 300 python tools/bench_c5.py --only 13:9:48:8,13:5:48:8,13:16:30:8 --max-batch-only > gpurun_out/r16/c5_2g_r$r.jsonl 2>/dev/null
timeout 300 python tools/bench_c5.py --only 13:9:48:8,13:5:48:8,13:16:30:8 --max-batch-only --one-team > gpurun_out/r16/c5_1t_r$r.jsonl 2>/dev/null
done
python3 -c "
import json,glob
for f in sorted(glob.glob('gpurun_out/r16/c5_*.jsonl')):
    for l in open(f):
        r=json.loads(l)
        if 'ntt_fwd' in r: print(f.split('/')[-1], r['log2N'],r['L'],r['bits'],r['batch'],r['ntt_fwd']['frac_hbm'],r['ntt_inv']['frac_hbm'],r['clocks'].get('sm_mhz'), r['clocks'].get('reasons'))
"
