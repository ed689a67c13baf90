mkdir -p gpurun_out/r19
timeout 900 python bench.py --config c1q3 --steps 12000 --warmup 100 > gpurun_out/r19/bench_c1q3.json 2> gpurun_out/r19/bench_c1q3.err
timeout 900 python bench.py --config c2 --steps 3000 --warmup 20 > gpurun_out/r19/bench_c2.json 2> gpurun_out/r19/bench_c2.err
timeout 900 python bench.py --config c3 --steps 60 --warmup 3 > gpurun_out/r19/bench_c3.json 2> gpurun_out/r19/bench_c3.err
timeout 900 python bench.py > gpurun_out/r19/bench_c4.json 2> gpurun_out/r19/bench_c4.err
python3 - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/r19/bench_*.json")):
    try:
        d = json.loads(open(f).readline())
        print(f.split("/")[-1], d["value"], d["ms_per_step"], d["steps"], d["clocks"], (d.get("e2e") or {}).get("value"), d["roofline"]["frac"])
    except Exception as e:
        print(f, "ERR", e)
PY
nvidia-smi --query-gpu=clocks.sm,power.draw,clocks_event_reasons.active --format=csv,noheader -lms 200 > gpurun_out/r19/fp64_ceiling_clocks.csv &
SMI=$!
./tools/int_peak sustained 4 > gpurun_out/r19/fp64_ceiling.json
kill $SMI
cat gpurun_out/r19/fp64_ceiling.json; sort gpurun_out/r19/fp64_ceiling_clocks.csv | uniq -c | sort -rn | head -5
./tools/int_peak > gpurun_out/r19/int_peak.jsonl
timeout 1500 python tools/bench_c5.py --points all > gpurun_out/r19/c5_all.jsonl 2> gpurun_out/r19/c5_all.err; wc -l gpurun_out/r19/c5_all.jsonl
ncu --set full --clock-control none --import-source on -k regex:k_ntt_c5 -c 1 -o gpurun_out/r19/fwd14_cl2g python tools/c5_point.py --lg 14 --L 9 --bits 48 --op fwd --batch 1024 --reps 1 > gpurun_out/r19/ncu1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_ntt_c5 -c 1 -o gpurun_out/r19/inv14_cl2g python tools/c5_point.py --lg 14 --L 9 --bits 48 --op inv --batch 1024 --reps 1 > gpurun_out/r19/ncu2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_ntt_c5 -c 1 -o gpurun_out/r19/inv13 python tools/c5_point.py --lg 13 --L 9 --bits 48 --op inv --batch 2048 --reps 1 > gpurun_out/r19/ncu3.log 2>&1
tail -n 1 gpurun_out/r19/ncu*.log
timeout 1200 python bench.py --config c4 --impl reference --threads 1 --steps 1 --warmup 1 > gpurun_out/r19/ref1_c4.json 2> gpurun_out/r19/ref1_c4.err; cat gpurun_out/r19/ref1_c4.json | cut -c1-300
