mkdir -p gpurun_out/r11
timeout 900 python -m pytest tests/test_gpu_find_dmax.py -x -q > gpurun_out/r11/pytest_dmax.log 2>&1; tail -3 gpurun_out/r11/pytest_dmax.log
timeout 2400 python tools/find_dmax.py --grid default --trials 1000 --dcap 8192 > gpurun_out/r11/dmax_default.jsonl 2> gpurun_out/r11/dmax_default.err; tail -3 gpurun_out/r11/dmax_default.err
cat gpurun_out/r11/dmax_default.jsonl | cut -c1-220
timeout 900 python tools/find_dmax.py --grid cap --trials 1000 --dcap 8192 > gpurun_out/r11/dmax_cap.jsonl 2> gpurun_out/r11/dmax_cap.err; tail -3 gpurun_out/r11/dmax_cap.err
cat gpurun_out/r11/dmax_cap.jsonl | cut -c1-220
