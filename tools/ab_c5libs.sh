#!/bin/bash
# A/B of libephdc.so builds (ablibs/lib<V>.so) on the c5 points: each build is copied over
# the in-tree library (the GPU box's scratch copy) before its runs; two rounds.
# usage: [LIBS="A B"] [POINTS="13:9:48:8 14:9:48:8"] tools/ab_c5libs.sh <tag>
O=gpurun_out/${1:-abc5}; mkdir -p $O
LIB=paper_2511_00737_b200/libephdc.so
cp $LIB $O/libephdc.orig.so
for r in 1 2; do
  for v in ${LIBS:-A B}; do
    cp ablibs/lib$v.so $LIB
    for p in ${POINTS:-13:9:48:8}; do
      timeout 300 python tools/bench_c5.py --only $p --max-batch-only $EXTRA > $O/${v}_${p//:/_}_r$r.jsonl 2>/dev/null
    done
  done
done
cp $O/libephdc.orig.so $LIB
python3 - "$O" <<'PY'
import glob, json, sys, os
for f in sorted(glob.glob(sys.argv[1] + "/*.jsonl")):
    for l in open(f):
        r = json.loads(l)
        if "ntt_fwd" in r:
            print(os.path.basename(f), r["log2N"], r["batch"], r["ntt_fwd"]["frac_hbm"], r["ntt_inv"]["frac_hbm"],
                  r["clocks"].get("sm_mhz"), r["clocks"].get("reasons"))
        elif r.get("op") == "mac":
            print(os.path.basename(f), "mac", r["log2N"], r["L"], r["bits"], r["D"], r["frac_hbm"],
                  r["clocks"].get("sm_mhz"), r["clocks"].get("reasons"))
PY
