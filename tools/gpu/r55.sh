mkdir -p gpurun_out/r55
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q -k "u64_words_30bit or bitexact or u32 or sampled" > gpurun_out/r55/pytest.log 2>&1; tail -n 3 gpurun_out/r55/pytest.log
timeout 900 python tools/bench_c5.py --points all --only 12:9:30:8,13:9:30:8,14:9:30:8,13:16:30:8,14:1:30:8 --max-batch-only > gpurun_out/r55/c5_30u64.jsonl 2> gpurun_out/r55/err.txt
python3 - <<'PY'
import json
for l in open("gpurun_out/r55/c5_30u64.jsonl"):
    d = json.loads(l)
    if "ntt_fwd" in d:
        print(d["log2N"], d["L"], d["batch"], d["ntt_fwd"]["frac_hbm"], d["ntt_inv"]["frac_hbm"], d["clocks"]["sm_mhz"], d["clocks"]["reasons"], d["kernels"])
PY
tail -n 3 gpurun_out/r55/err.txt
