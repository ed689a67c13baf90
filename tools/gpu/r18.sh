mkdir -p gpurun_out/r18
timeout 300 python tools/bench_c5.py --only 15:5:48:8 --max-batch-only > gpurun_out/r18/c5_15.jsonl 2> gpurun_out/r18/c5_15.err; tail -n 3 gpurun_out/r18/c5_15.err; cat gpurun_out/r18/c5_15.jsonl | cut -c1-300
timeout 300 python tools/bench_c5.py --only 16:3:48:8 --max-batch-only > gpurun_out/r18/c5_16.jsonl 2> gpurun_out/r18/c5_16.err; tail -n 3 gpurun_out/r18/c5_16.err; cat gpurun_out/r18/c5_16.jsonl | cut -c1-300
ncu --set full --clock-control none --import-source on -k regex:k_ntt_mac_f64 -c 1 -o gpurun_out/r18/c4_2g python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/r18/ncu1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_ntt_mac_f64 -c 1 -o gpurun_out/r18/c4_1t python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e --plan flags=32 > gpurun_out/r18/ncu2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_ntt_mac_f64 -c 1 -o gpurun_out/r18/c3_2g python bench.py --config c3 --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/r18/ncu3.log 2>&1
tail -n 1 gpurun_out/r18/ncu*.log
