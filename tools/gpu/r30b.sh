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
ncu --set full --clock-control none -k regex:k_ntt_batch -c 1 -o /tmp/u32fwd13 python /tmp/u32.py 13 fwd > /dev/null 2>&1
ncu --set full --clock-control none -k regex:k_ntt_batch -c 1 -o /tmp/u32inv13 python /tmp/u32.py 13 inv > /dev/null 2>&1
ncu --set full --clock-control none -k regex:k_mac -c 1 -o /tmp/mac48 python tools/c5_point.py --lg 13 --L 9 --bits 48 --op mac --reps 1 > /dev/null 2>&1
ncu --set full --clock-control none -k regex:k_pack_intt_q -c 1 -o /tmp/pack_c4 python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e > /dev/null 2>&1
for k in u32fwd13 u32inv13 mac48 pack_c4; do python tools/ncu_brief.py /tmp/$k.ncu-rep > gpurun_out/r30/ncu_$k.txt 2>&1; done
ls -la gpurun_out/r30/
