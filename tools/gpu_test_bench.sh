#!/bin/bash
# One gpurun call: GPU tests + bench lines (no profiler).
# usage: tools/gpu_test_bench.sh <tag> [configs...]
TAG=${1:-v}; shift; CFGS=${@:-c4}
O=gpurun_out/$TAG; mkdir -p $O
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/rc.txt
timeout 1500 python -m pytest tests -m gpu -x -q -rA --durations=15 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
for c in $CFGS; do
  timeout 900 python bench.py --config $c > $O/bench_$c.json 2> $O/bench_$c.err; echo "bench $c rc=$?" >> $O/rc.txt
done
