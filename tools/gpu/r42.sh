mkdir -p gpurun_out/r42
timeout 900 python tools/bench_c5.py --points all --only 12:9:30:4,13:9:30:4,14:9:30:4,13:1:30:4,14:16:30:4 --max-batch-only > gpurun_out/r42/c5u32.jsonl 2> gpurun_out/r42/c5u32.err; tail -n 3 gpurun_out/r42/c5u32.err
timeout 600 python tools/bench_c5.py --points all --only 12:9:30:4,13:9:30:4,14:9:30:4 --max-batch-only --u32-generic > gpurun_out/r42/c5u32_gen.jsonl 2>> gpurun_out/r42/c5u32.err
python3 - <<'PY'
import json
for f in ("gpurun_out/r42/c5u32.jsonl", "gpurun_out/r42/c5u32_gen.jsonl"):
    for l in open(f):
        d = json.loads(l)
        if "ntt_fwd" in d:
            print(f.split("/")[-1], d["log2N"], d["L"], d["batch"], d["ntt_fwd"]["frac_hbm"], d["ntt_inv"]["frac_hbm"], d["clocks"]["sm_mhz"], d["clocks"]["reasons"], d["kernels"])
PY
for op in fwd inv; do
timeout 300 python tools/c5_point.py --lg 13 --L 9 --bits 30 --op $op --u32 --reps 3 > gpurun_out/r42/pt13_$op.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_ntt32_c5 -s 2 -c 1 -o gpurun_out/r42/ncu_u32_${op}13 python tools/c5_point.py --lg 13 --L 9 --bits 30 --op $op --u32 --reps 3 > gpurun_out/r42/ncu_${op}13.log 2>&1; tail -n 2 gpurun_out/r42/ncu_${op}13.log
done
