mkdir -p gpurun_out/r20
for spec in "14 5 30 fwd 52428" "14 5 30 inv 52428" "14 5 48 fwd 52428" "14 5 48 inv 52428" "14 5 30 fwd 16384" "14 5 30 inv 16384" "14 9 30 fwd 29127" "14 9 30 inv 29127" "14 5 30 fwd 4096" "14 1 30 fwd 65536" "14 1 30 inv 65536"; do
  set -- $spec
  echo -n "$spec: "
  timeout 120 python tools/c5_point.py --lg $1 --L $2 --bits $3 --op $4 --batch $5 --reps 2 2>&1 | tail -n 1 | cut -c1-150
done
python3 -c "
import paper_2511_00737_b200 as eph
for bits in (30, 48):
    q = eph.find_ntt_primes(14, [bits]*5); p = eph.NttPlan(q, 14); print(bits, p.fwd_kernel, p.inv_kernel)
"
