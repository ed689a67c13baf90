mkdir -p gpurun_out/r14
LIBS="A B C D" POINTS="13:9:48:8 14:9:48:8" bash tools/ab_c5libs.sh r14/ab
timeout 600 python bench.py --no-cpu > gpurun_out/r14/bench.json 2> gpurun_out/r14/bench.err; python3 -c "import json; d=json.loads(open('gpurun_out/r14/bench.json').readline()); print(d['value'], d['ms_per_step'], d['roofline']['kernel_ms'], d['clocks'])"
