mkdir -p gpurun_out/r22
for spec in "14 3 48 fwd 65536" "14 3 48 inv 65536" "16 9 30 fwd 7281" "16 9 30 inv 7281" "15 5 48 fwd 26214" "15 5 48 inv 26214"; do
  set -- $spec
  for rep in 1 2 3; do
    echo -n "$spec rep$rep: "
    timeout 120 python tools/c5_point.py --lg $1 --L $2 --bits $3 --op $4 --batch $5 --reps 100 2>&1 | tail -n 1 | cut -c1-120
  done
done
