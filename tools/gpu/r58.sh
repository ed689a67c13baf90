O=gpurun_out/r58; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q -k "u64_words_30bit or u32" > $O/pytest.log 2>&1; tail -n 2 $O/pytest.log
timeout 900 python -m pytest tests/test_gpu_c5_sweep.py -x -q -k "30b" > $O/pytest_sweep30.log 2>&1; tail -n 2 $O/pytest_sweep30.log
timeout 900 python tools/bench_c5.py --points all --only 12:9:30:4,13:9:30:4,14:9:30:4,12:9:30:8,13:9:30:8,14:9:30:8 --max-batch-only > $O/c5_30.jsonl 2> $O/err.txt
python3 - <<'PY'
import json
for l in open("gpurun_out/r58/c5_30.jsonl"):
    d = json.loads(l)
    if "ntt_fwd" in d:
        print(d["log2N"], d["word_bits"], d["batch"], d["ntt_fwd"]["frac_hbm"], d["ntt_inv"]["frac_hbm"], d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
PY
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_encode_tc|k_pack_intt|k_ntt_mac_f64" -s 6 -c 3 -o $O/c4 $CMD > $O/ncu_full.log 2>&1; echo "full rc=$?"
