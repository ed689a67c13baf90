LIBS="BASE PRE1 PRE3 TMO PRE1TMO" bash tools/ab_libs.sh r31 c4
python3 - <<'PY'
import json, glob, os
for f in sorted(glob.glob("gpurun_out/r31/c4_*.json")):
    try:
        d = json.loads(open(f).readline())
        print(os.path.basename(f), d["value"], d["roofline"]["kernel_ms"]["ntt_mac"], d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
    except Exception as e:
        print(f, "ERR", e)
PY
