mkdir -p gpurun_out/r8
timeout 2400 python -m pytest tests/test_gpu_c5_sweep.py tests/test_gpu_fullsize.py -x -q --durations=15 > gpurun_out/r8/pytest_slow.log 2>&1; tail -25 gpurun_out/r8/pytest_slow.log
timeout 1800 python tools/bench_c5.py --points all > gpurun_out/r8/bench_c5_all.jsonl 2> gpurun_out/r8/bench_c5.err; wc -l gpurun_out/r8/bench_c5_all.jsonl; tail -3 gpurun_out/r8/bench_c5.err
timeout 600 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/r8/b.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_ntt_mac_f64|k_pack_intt_q|k_encode_tc" -s 3 -c 3 -o gpurun_out/r8/c4 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/r8/ncu.log 2>&1; tail -3 gpurun_out/r8/ncu.log
