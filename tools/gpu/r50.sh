mkdir -p gpurun_out/r50
timeout 1500 python -m pytest tests/test_gpu_variants.py tests/test_gpu_parity.py -x -q > gpurun_out/r50/pytest.log 2>&1; tail -n 2 gpurun_out/r50/pytest.log
for r in 1 2; do
for v in "" "flags=256" "flags=128"; do
  tag=${v:-default}; tag=${tag/=/}
  timeout 600 python bench.py --no-e2e --no-cpu ${v:+--plan $v} > gpurun_out/r50/c4_${tag}_r$r.json 2> gpurun_out/r50/err_${tag}_r$r.txt
  python3 -c "import json; d=json.loads(open('gpurun_out/r50/c4_${tag}_r$r.json').readline()); print('$tag', $r, d['value'], d['roofline']['kernel_ms'], d['clocks']['sm_mhz'])"
done; done
for c in c3 c2; do for v in "" "flags=256"; do tag=${v:-default}; tag=${tag/=/}
  timeout 600 python bench.py --config $c --no-e2e --no-cpu ${v:+--plan $v} > gpurun_out/r50/${c}_${tag}.json 2>> gpurun_out/r50/err.txt
  python3 -c "import json; d=json.loads(open('gpurun_out/r50/${c}_${tag}.json').readline()); print('$c $tag', d['value'], d['roofline']['kernel_ms'])"
done; done
