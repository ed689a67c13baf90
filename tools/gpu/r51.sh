mkdir -p gpurun_out/r51
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_sr.py -x -q -k "mac or sr" > gpurun_out/r51/pytest_mac.log 2>&1; tail -n 2 gpurun_out/r51/pytest_mac.log
timeout 900 python -m pytest tests/test_gpu_c5_sweep.py -x -q -k "60b" > gpurun_out/r51/pytest_sweep60.log 2>&1; tail -n 2 gpurun_out/r51/pytest_sweep60.log
timeout 900 python tools/bench_c5.py --points all --only 12:9:60:8,13:9:60:8,14:9:60:8,13:16:60:8 --max-batch-only > gpurun_out/r51/c5_60.jsonl 2> gpurun_out/r51/err.txt
python3 - <<'PY'
import json
for l in open("gpurun_out/r51/c5_60.jsonl"):
    d = json.loads(l)
    if d.get("op") == "mac":
        print("mac", d["log2N"], d["L"], d["D"], d["frac_hbm"], d["clocks"]["sm_mhz"])
PY
tail -n 3 gpurun_out/r51/err.txt
