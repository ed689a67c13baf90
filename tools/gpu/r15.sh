# measurement hygiene run: every config's bench line (clocks, cpu_baseline all cores), the
# single-core oracle for c1q3-c3, the oracle reference arm at c4, SR with clocks, c5 sweep
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q > gpurun_out/r15/pytest_k.log 2>&1; tail -n 2 gpurun_out/r15/pytest_k.log
mkdir -p gpurun_out/r15
for c in c1q3 c2 c3 c4; do
  timeout 900 python bench.py --config $c > gpurun_out/r15/bench_$c.json 2> gpurun_out/r15/bench_$c.err
done
for c in c1q3 c2 c3; do
  timeout 900 python bench.py --config $c --impl reference --threads 1 --steps 3 --warmup 1 > gpurun_out/r15/ref1_$c.json 2> gpurun_out/r15/ref1_$c.err
done
timeout 900 python bench.py --config c4 --impl reference --steps 5 --warmup 3 > gpurun_out/r15/ref_c4.json 2> gpurun_out/r15/ref_c4.err
timeout 900 python tools/bench_sr.py --configs c2 c3 c4 > gpurun_out/r15/sr.jsonl 2> gpurun_out/r15/sr.err
timeout 1500 python tools/bench_c5.py --points all > gpurun_out/r15/c5_all.jsonl 2> gpurun_out/r15/c5_all.err
python3 - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/r15/*.json")):
    try:
        d = json.loads(open(f).readline())
    except Exception as e:
        print(f, "ERR", e); continue
    print(f.split("/")[-1], d.get("value"), d.get("ms_per_step"), d.get("steps"), (d.get("clocks") or {}).get("sm_mhz"),
          (d.get("cpu_baseline") or {}).get("value"), (d.get("e2e") or {}).get("value"))
PY
wc -l gpurun_out/r15/c5_all.jsonl gpurun_out/r15/sr.jsonl
