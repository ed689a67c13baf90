mkdir -p gpurun_out/r47
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q -k "u32" > gpurun_out/r47/pytest_u32.log 2>&1; tail -n 2 gpurun_out/r47/pytest_u32.log
for r in 1 2; do
timeout 900 python tools/bench_c5.py --points all --only 12:9:30:4,13:9:30:4 --max-batch-only > gpurun_out/r47/def_$r.jsonl 2> gpurun_out/r47/err.txt
timeout 900 python tools/bench_c5.py --points all --only 12:9:30:4,13:9:30:4 --max-batch-only --alt-teams > gpurun_out/r47/occ_$r.jsonl 2>> gpurun_out/r47/err.txt
done
python3 - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/r47/*.jsonl")):
    for l in open(f):
        d = json.loads(l)
        if "ntt_fwd" in d:
            print(f.split("/")[-1], d["log2N"], d["L"], d["batch"], d["ntt_fwd"]["frac_hbm"], d["ntt_inv"]["frac_hbm"], d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
PY
tail -n 3 gpurun_out/r47/err.txt
