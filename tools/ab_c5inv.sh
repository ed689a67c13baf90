#!/bin/bash
# c5 FP64 cluster inverse: split-barrier kernel (default) vs the unsplit one (--alt-teams), tests first
O=gpurun_out/${1:-r65}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_kernels.py -m gpu -x -q > $O/pytest_kernels.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
P=14:9:48:8,15:5:48:8,16:5:48:8,14:5:48:8,14:16:48:8
for r in 1 2; do
  timeout 600 python tools/bench_c5.py --only $P --max-batch-only > $O/c5inv_new_$r.jsonl 2> $O/c5inv_new_$r.err; echo "new $r rc=$?" >> $O/rc.txt
  timeout 600 python tools/bench_c5.py --only $P --max-batch-only --alt-teams > $O/c5inv_old_$r.jsonl 2> $O/c5inv_old_$r.err; echo "old $r rc=$?" >> $O/rc.txt
done
