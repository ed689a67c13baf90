mkdir -p gpurun_out/r28
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -k "u32 or prime_switch" > gpurun_out/r28/pytest_k.log 2>&1; tail -n 2 gpurun_out/r28/pytest_k.log
timeout 900 python -m pytest tests/test_gpu_c5_sweep.py -x -q -k "u32" > gpurun_out/r28/pytest_sweep.log 2>&1; tail -n 2 gpurun_out/r28/pytest_sweep.log
for r in 1 2; do
timeout 300 python tools/bench_c5.py --points all --only 12:9:30:4,13:9:30:4,12:16:30:4,13:16:30:4,13:1:30:4 --max-batch-only > gpurun_out/r28/u32_2g_r$r.jsonl 2>/dev/null
timeout 300 python tools/bench_c5.py --points all --only 12:9:30:4,13:9:30:4,12:16:30:4,13:16:30:4,13:1:30:4 --max-batch-only --alt-teams > gpurun_out/r28/u32_alt_r$r.jsonl 2>/dev/null
done
python3 -c "
import json,glob
for f in sorted(glob.glob('gpurun_out/r28/u32_*.jsonl')):
    for l in open(f):
        r=json.loads(l)
        if 'ntt_fwd' in r: print(f.split('/')[-1], r['log2N'],r['L'],r['bits'],r['word_bits'],r['batch'],r['ntt_fwd']['frac_hbm'],r['ntt_inv']['frac_hbm'],r['clocks'].get('sm_mhz'))
"
