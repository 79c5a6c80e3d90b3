#!/bin/bash
# attention backward tail split (DPL_ATTN_BWD_SPLIT=1 default) vs off, same build
out=gpurun_out/r2attntail; mkdir -p $out
timeout 900 python -m pytest tests/test_attention_gpu.py tests/test_executor_gpu.py tests/test_baseline_shapes_gpu.py -m gpu -q -x --timeout 300 --timeout-method thread -p no:cacheprovider -rf > $out/pytest.txt 2>&1
tail -1 $out/pytest.txt
for v in 1 0 1 0; do echo "== split=$v"; DPL_ATTN_BWD_SPLIT=$v timeout 120 python tools/attn_bench.py 2>&1 | tail -4; done
for v in 1 0 1 0; do
  DPL_ATTN_BWD_SPLIT=$v timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e > $out/bert_$v.json 2> $out/bert_$v.err
  python -c "import json; d=json.load(open('$out/bert_$v.json')); print('bert split=$v', round(d['value'],2), d['clocks']['sm_mhz'], round(d['roofline']['frac'],4), [(k['kernel'], round(k['seconds']*1e3,2), round(k.get('tflops',0))) for k in d['kernels'] if 'attention' in k['kernel']])"
done
for v in 1 0; do
  DPL_ATTN_BWD_SPLIT=$v timeout 600 python bench.py --model xlnet36 --steps 3 --warmup 3 --no-cpu --no-e2e > $out/xlnet_$v.json 2> $out/xlnet_$v.err
  python -c "import json; d=json.load(open('$out/xlnet_$v.json')); print('xlnet split=$v', round(d['value'],2), d['clocks']['sm_mhz'])"
done
