mkdir -p gpurun_out/r41
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q -k "u32" > gpurun_out/r41/pytest_u32.log 2>&1; tail -n 3 gpurun_out/r41/pytest_u32.log
timeout 600 python tools/bench_c5.py --only 12:9:30:4,13:9:30:4,14:9:30:4,13:1:30:4,14:16:30:4 --max-batch-only > gpurun_out/r41/c5u32.jsonl 2> gpurun_out/r41/c5u32.err; tail -n 3 gpurun_out/r41/c5u32.err
timeout 600 python tools/bench_c5.py --only 12:9:30:4,13:9:30:4,14:9:30:4 --max-batch-only --u32-generic > gpurun_out/r41/c5u32_gen.jsonl 2>> gpurun_out/r41/c5u32.err
python3 - <<'PY'
import json
for f in ("gpurun_out/r41/c5u32.jsonl", "gpurun_out/r41/c5u32_gen.jsonl"):
    for l in open(f):
        d = json.loads(l)
        if "ntt_fwd" in d:
            print(f.split("/")[-1], d["log2N"], d["L"], d["batch"], d["ntt_fwd"]["frac_hbm"], d["ntt_inv"]["frac_hbm"], d["clocks"]["sm_mhz"], d["clocks"]["reasons"], d["kernels"])
PY
timeout 900 python -m pytest tests/test_gpu_c5_sweep.py -x -q -k "u32" > gpurun_out/r41/pytest_sweep_u32.log 2>&1; tail -n 3 gpurun_out/r41/pytest_sweep_u32.log
