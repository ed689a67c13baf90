mkdir -p gpurun_out/r24
for spec in "14 3 48 fwd 65536" "14 3 48 inv 65536" "16 9 30 fwd 7281" "16 9 30 inv 7281" "15 5 48 fwd 26214" "15 5 48 inv 26214" "14 9 48 fwd 29127"; do
  set -- $spec
  for rep in 1 2 3; do
    echo -n "$spec rep$rep: "
    timeout 120 python tools/c5_point.py --lg $1 --L $2 --bits $3 --op $4 --batch $5 --reps 100 2>&1 | tail -n 1 | cut -c1-120
  done
done
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q > gpurun_out/r24/pytest_k.log 2>&1; tail -n 2 gpurun_out/r24/pytest_k.log
timeout 1500 python -m pytest tests/test_gpu_c5_sweep.py -x -q > gpurun_out/r24/pytest_sweep.log 2>&1; tail -n 2 gpurun_out/r24/pytest_sweep.log
for r in 1 2; do
timeout 300 python tools/bench_c5.py --points all --only 12:9:30:4,13:9:30:4,14:9:30:4,12:9:60:8,13:9:60:8,13:16:30:4,12:16:30:4 --max-batch-only > gpurun_out/r24/int_new_r$r.jsonl 2>/dev/null
timeout 300 python tools/bench_c5.py --points all --only 12:9:30:4,13:9:30:4,14:9:30:4,12:9:60:8,13:9:60:8,13:16:30:4,12:16:30:4 --max-batch-only --alt-teams > gpurun_out/r24/int_alt_r$r.jsonl 2>/dev/null
done
python3 -c "
import json,glob
for f in sorted(glob.glob('gpurun_out/r24/int_*.jsonl')):
    for l in open(f):
        r=json.loads(l)
        if 'ntt_fwd' in r: print(f.split('/')[-1], r['log2N'],r['L'],r['bits'],r['word_bits'],r['batch'],r['ntt_fwd']['frac_hbm'],r['ntt_inv']['frac_hbm'],r['kernels'],r['clocks'].get('sm_mhz'))
"
