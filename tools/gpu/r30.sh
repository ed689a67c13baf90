mkdir -p gpurun_out/r30
cat > /tmp/u32.py <<'PY'
import sys, os
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import torch, paper_2511_00737_b200 as eph
lg = int(sys.argv[1]); op = sys.argv[2]
q = eph.find_ntt_primes(lg, [30] * 9); plan = eph.NttPlan(q, lg)
x = torch.randint(0, 1 << 29, (2048, 9, 1 << lg), dtype=torch.int32, device="cuda")
f = eph.ntt_fwd32 if op == "fwd" else eph.ntt_inv32
f(plan, x); torch.cuda.synchronize()
PY
ncu --set full --clock-control none -k regex:k_ntt_batch -c 1 -o gpurun_out/r30/u32fwd13 python /tmp/u32.py 13 fwd > gpurun_out/r30/ncu1.log 2>&1
ncu --set full --clock-control none -k regex:k_ntt_batch -c 1 -o gpurun_out/r30/u32inv13 python /tmp/u32.py 13 inv > gpurun_out/r30/ncu2.log 2>&1
ncu --set full --clock-control none -k regex:k_mac -c 1 -o gpurun_out/r30/mac48 python tools/c5_point.py --lg 13 --L 9 --bits 48 --op mac --reps 1 > gpurun_out/r30/ncu3.log 2>&1
ncu --set full --clock-control none -k regex:k_pack_intt_q -c 1 -o gpurun_out/r30/pack_c4 python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/r30/ncu4.log 2>&1
tail -n 1 gpurun_out/r30/ncu*.log
