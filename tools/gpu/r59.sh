O=gpurun_out/r59; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_variants.py tests/test_gpu_parity.py -x -q > $O/pytest.log 2>&1; tail -n 2 $O/pytest.log
for r in 1 2; do for v in "" "flags=256"; do tag=${v:-pf}; tag=${tag/=/}
  timeout 600 python bench.py --no-e2e --no-cpu ${v:+--plan $v} > $O/c4_${tag}_r$r.json 2> $O/err.txt
  python3 -c "import json; d=json.loads(open('$O/c4_${tag}_r$r.json').readline()); print('$tag', $r, d['value'], d['roofline']['kernel_ms'], d['clocks']['sm_mhz'])"
done; done
for v in "" "flags=256"; do tag=${v:-pf}; tag=${tag/=/}
  timeout 600 python bench.py --config c3 --no-e2e --no-cpu ${v:+--plan $v} > $O/c3_${tag}.json 2>> $O/err.txt
  python3 -c "import json; d=json.loads(open('$O/c3_${tag}.json').readline()); print('c3 $tag', d['value'], d['roofline']['kernel_ms'])"
done
