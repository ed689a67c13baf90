#!/bin/bash
# One gpurun call: smoke, GPU tests, bench and ONE ncu pass -- the launch list (NCU=launch,
# default) or the --set full capture of the top kernel (NCU=full).
# usage: [NCU=launch|full] tools/gpu_profile_round.sh <tag> [config] [kernel-regex]
TAG=${1:-v}; CFG=${2:-c4}; KRE=${3:-k_ntt_mac}
O=gpurun_out/$TAG; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $O/smi.txt 2>&1
(nproc; lscpu | grep -E 'Model name|^CPU\(s\)') > $O/host.txt 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/rc.txt
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
timeout 900 python bench.py --config $CFG > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/rc.txt
CMD="python bench.py --config $CFG --steps 1 --warmup 3 --no-e2e --no-cpu"
timeout 600 $CMD > $O/plain.log 2>&1 && echo "plain rc=0" >> $O/rc.txt && \
if [ "${NCU:-launch}" = full ]; then
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:$KRE -s 3 -c 1 -o $O/prof $CMD > $O/ncu_full.log 2>&1
else
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv $CMD > $O/ncu_launch.log 2>&1
fi; echo "ncu rc=$?" >> $O/rc.txt
