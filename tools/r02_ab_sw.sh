#!/bin/bash
# residual / activation-input GEMMs: 2 prefetched input chunks per warp (default, 4 ring stages)
# vs 1 chunk (DPL_GEMM_X_BUFS=1, 5 stages)
out=gpurun_out/r2abxb; mkdir -p $out
timeout 600 python -m pytest tests/test_gemm_gpu.py -m gpu -q -x --timeout 300 --timeout-method thread -p no:cacheprovider > $out/pytest.txt 2>&1; tail -1 $out/pytest.txt
for r in 1 2; do for v in 2 1; do
  DPL_GEMM_X_BUFS=$v timeout 200 python tools/gemm_graph_bench.py > $out/gg_$v_$r.txt 2>&1
  echo "xbufs=$v $(python - <<PY
import json
for l in open('$out/gg_$v_$r.txt'):
    l=l.strip()
    if not l.startswith('{'): continue
    d=json.loads(l)
    if 'gemm' in d and d['gemm'] in ('o','ffn2','o_dgrad','ffn1_dgrad','qkv_dgrad'): print(d['gemm'], d['ours_us'], end='; ')
    if 'sum_us' in d: print('sum', d['sum_us']['ours'])
PY
)"
  for m in bert48 gpt2-1.5b; do
    DPL_GEMM_X_BUFS=$v timeout 600 python bench.py --model $m --steps 5 --warmup 3 --no-cpu > $out/${m}_$v_$r.json 2>/dev/null
    echo "  $m xbufs=$v $(python -c "import json; d=json.load(open('$out/${m}_$v_$r.json')); print(round(d['value'],2), d['clocks']['sm_mhz'])" 2>&1 | tail -1)"
  done
done; done
