mkdir -p gpurun_out/r27
EXTRA="--points all" LIBS="OLD NEW" POINTS="14:3:48:8 14:9:48:8 15:5:48:8 16:3:48:8" bash tools/ab_c5libs.sh r27/ab | grep -v mac
timeout 900 python tools/bench_sr.py --configs c2 c3 c4 > gpurun_out/r27/sr.jsonl 2> gpurun_out/r27/sr.err; cut -c1-200 gpurun_out/r27/sr.jsonl
cat > /tmp/u32.py <<'PY'
import sys, torch, paper_2511_00737_b200 as eph
lg = int(sys.argv[1]); op = sys.argv[2]
q = eph.find_ntt_primes(lg, [30] * 9); plan = eph.NttPlan(q, lg)
x = torch.randint(0, 1 << 29, (2048, 9, 1 << lg), dtype=torch.int32, device="cuda")
f = eph.ntt_fwd32 if op == "fwd" else eph.ntt_inv32
f(plan, x); torch.cuda.synchronize()
PY
ncu --set full --clock-control none --import-source on -k regex:k_ntt_batch -c 1 -o gpurun_out/r27/u32fwd13 python /tmp/u32.py 13 fwd > gpurun_out/r27/ncu1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_ntt_batch -c 1 -o gpurun_out/r27/u32inv13 python /tmp/u32.py 13 inv > gpurun_out/r27/ncu2.log 2>&1
tail -n 1 gpurun_out/r27/ncu*.log
