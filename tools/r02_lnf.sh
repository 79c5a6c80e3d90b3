#!/bin/bash
# LayerNorm forward: 2 rows per warp (default) vs 1 (DPL_LN_FWD_ROWS=1)
out=gpurun_out/r2lnf; mkdir -p $out
timeout 600 python -m pytest tests/test_elementwise_gpu.py tests/test_executor_gpu.py -m gpu -q -x --timeout 300 --timeout-method thread -p no:cacheprovider > $out/pytest.txt 2>&1; tail -1 $out/pytest.txt
for v in 2 1 2 1; do echo "== rows=$v"; DPL_LN_FWD_ROWS=$v timeout 120 python tools/elementwise_graph_bench.py 2>&1 | grep layernorm_fwd; done
for v in 2 1 2 1; do
  DPL_LN_FWD_ROWS=$v timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e > $out/bert_$v.json 2> $out/bert_$v.err
  python -c "import json; d=json.load(open('$out/bert_$v.json')); print('bert rows=$v', round(d['value'],2), d['clocks']['sm_mhz'], [(k['kernel'], round(k['seconds']*1e3,2)) for k in d['kernels'] if 'layernorm' in k['kernel']])"
done
