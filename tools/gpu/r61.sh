O=gpurun_out/r61; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q -k "u32 or u64_words_30bit" > $O/pytest.log 2>&1; tail -n 2 $O/pytest.log
timeout 900 python -m pytest tests/test_gpu_c5_sweep.py -x -q -k "u32" > $O/pytest_sweep.log 2>&1; tail -n 2 $O/pytest_sweep.log
timeout 900 python tools/bench_c5.py --points all --only 15:9:30:4,16:9:30:4,14:9:30:4,13:9:30:4,12:9:30:4,13:9:30:8,14:9:30:8 --max-batch-only > $O/c5u32.jsonl 2> $O/err.txt
python3 - <<'PY'
import json
for l in open("gpurun_out/r61/c5u32.jsonl"):
    d = json.loads(l)
    if "ntt_fwd" in d:
        print(d["log2N"], d["L"], d["batch"], d["ntt_fwd"]["frac_hbm"], d["ntt_inv"]["frac_hbm"], d["clocks"]["sm_mhz"], d["clocks"]["reasons"], d["kernels"])
PY
tail -n 3 $O/err.txt
