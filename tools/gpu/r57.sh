O=gpurun_out/r57; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q -k "u64_words_30bit or u32 or bitexact" > $O/pytest.log 2>&1; tail -n 2 $O/pytest.log
timeout 900 python -m pytest tests/test_gpu_c5_sweep.py -x -q -k "30b" > $O/pytest_sweep30.log 2>&1; tail -n 2 $O/pytest_sweep30.log
for r in 1 2; do
timeout 900 python tools/bench_c5.py --points all --only 12:9:30:4,13:9:30:4,14:9:30:4,12:9:30:8,13:9:30:8,14:9:30:8 --max-batch-only > $O/new_$r.jsonl 2> $O/err.txt
timeout 900 python tools/bench_c5.py --points all --only 12:9:30:4,13:9:30:4,14:9:30:4 --max-batch-only --alt-teams > $O/tma_$r.jsonl 2>> $O/err.txt
done
python3 - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/r57/*.jsonl")):
    for l in open(f):
        d = json.loads(l)
        if "ntt_fwd" in d:
            print(f.split("/")[-1], d["log2N"], d["word_bits"], d["batch"], d["ntt_fwd"]["frac_hbm"], d["ntt_inv"]["frac_hbm"], d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
PY
tail -n 3 $O/err.txt
