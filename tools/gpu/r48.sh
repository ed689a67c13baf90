mkdir -p gpurun_out/r48
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_c5_sweep.py -x -q -k "u32" > gpurun_out/r48/pytest_u32.log 2>&1; tail -n 2 gpurun_out/r48/pytest_u32.log
timeout 900 python tools/bench_c5.py --points all --only 12:9:30:4,13:9:30:4,14:9:30:4,13:16:30:4,14:1:30:4 --max-batch-only > gpurun_out/r48/c5u32.jsonl 2> gpurun_out/r48/err.txt
python3 - <<'PY'
import json
for l in open("gpurun_out/r48/c5u32.jsonl"):
    d = json.loads(l)
    if "ntt_fwd" in d:
        print(d["log2N"], d["L"], d["batch"], d["ntt_fwd"]["frac_hbm"], d["ntt_inv"]["frac_hbm"], d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
    else:
        print("mac", d["log2N"], d["L"], d["D"], d["frac_hbm"], d["clocks"]["sm_mhz"])
PY
tail -n 3 gpurun_out/r48/err.txt
