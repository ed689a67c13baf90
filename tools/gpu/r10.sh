mkdir -p gpurun_out/r10
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q > gpurun_out/r10/pytest_k.log 2>&1; tail -3 gpurun_out/r10/pytest_k.log
timeout 900 python -m pytest tests/test_gpu_c5_sweep.py -x -q -k "N32768 or N65536" > gpurun_out/r10/pytest_sweep.log 2>&1; tail -3 gpurun_out/r10/pytest_sweep.log
timeout 600 python tools/bench_c5.py --points quick --max-batch-only > gpurun_out/r10/c5_quick.jsonl 2> gpurun_out/r10/c5_quick.err
python3 -c "
import json
for l in open('gpurun_out/r10/c5_quick.jsonl'):
    r=json.loads(l)
    if 'ntt_fwd' in r: print(r['log2N'],r['L'],r['bits'],r['word_bits'],r['batch'],r['ntt_fwd']['frac_hbm'],r['ntt_inv']['frac_hbm'],r['kernels'],r['clocks'].get('sm_mhz'))
    else: print('mac',r['log2N'],r['L'],r['bits'],r['D'],r['frac_hbm'],r['clocks'].get('sm_mhz'))
"
timeout 120 python tools/c5_point.py --lg 13 --L 9 --bits 48 --op mac --reps 3 && \
ncu --set full --clock-control none -k regex:k_mac -c 1 -o gpurun_out/r10/mac48 python tools/c5_point.py --lg 13 --L 9 --bits 48 --op mac --reps 1 > gpurun_out/r10/ncu1.log 2>&1
ncu --set full --clock-control none -k regex:k_mac -c 1 -o gpurun_out/r10/mac30 python tools/c5_point.py --lg 13 --L 9 --bits 30 --op mac --reps 1 > gpurun_out/r10/ncu2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_ntt_c5 -c 1 -o gpurun_out/r10/fwd14 python tools/c5_point.py --lg 14 --L 9 --bits 48 --op fwd --batch 1024 --reps 1 > gpurun_out/r10/ncu3.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_ntt_c5 -c 1 -o gpurun_out/r10/fwd13 python tools/c5_point.py --lg 13 --L 9 --bits 48 --op fwd --batch 2048 --reps 1 > gpurun_out/r10/ncu4.log 2>&1
tail -n 1 gpurun_out/r10/ncu*.log
