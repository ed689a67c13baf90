mkdir -p gpurun_out/r13
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q > gpurun_out/r13/pytest_k.log 2>&1; tail -n 3 gpurun_out/r13/pytest_k.log
for lg in 13; do for b in 48 30; do
timeout 300 python tools/bench_c5.py --only $lg:9:$b:8 --max-batch-only > gpurun_out/r13/c5_2g_${b}.jsonl 2>/dev/null
timeout 300 python tools/bench_c5.py --only $lg:9:$b:8 --max-batch-only --one-team > gpurun_out/r13/c5_1t_${b}.jsonl 2>/dev/null
done; done
python3 -c "
import json,glob
for f in sorted(glob.glob('gpurun_out/r13/c5_*.jsonl')):
    for l in open(f):
        r=json.loads(l)
        if 'ntt_fwd' in r: print(f.split('/')[-1], r['log2N'],r['L'],r['bits'],r['batch'],r['ntt_fwd']['frac_hbm'],r['ntt_inv']['frac_hbm'],r['clocks'].get('sm_mhz'), r['clocks'].get('reasons'))
"
timeout 600 python bench.py --no-cpu > gpurun_out/r13/bench_a.json 2> gpurun_out/r13/bench_a.err; python3 -c "import json; d=json.loads(open('gpurun_out/r13/bench_a.json').readline()); print(d['value'], d['ms_per_step'], d['roofline']['kernel_ms'], d['clocks'])"
ncu --set full --clock-control none --import-source on -k regex:k_ntt_c5 -c 1 -o gpurun_out/r13/fwd13_2g python tools/c5_point.py --lg 13 --L 9 --bits 48 --op fwd --batch 2048 --reps 1 > gpurun_out/r13/ncu1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_ntt_c5 -c 1 -o gpurun_out/r13/inv13_2g python tools/c5_point.py --lg 13 --L 9 --bits 48 --op inv --batch 2048 --reps 1 > gpurun_out/r13/ncu2.log 2>&1
tail -n 1 gpurun_out/r13/ncu*.log
