#!/bin/bash
out=gpurun_out/r2attn4; mkdir -p $out
timeout 600 python -m pytest tests/test_attention_gpu.py tests/test_lm_gpu.py -m gpu -q -x --timeout 300 --timeout-method thread -p no:cacheprovider -rf > $out/pytest_attn.txt 2>&1
tail -1 $out/pytest_attn.txt
timeout 120 python tools/attn_trace.py 8 512 16 0 > $out/trace_bert.txt 2>&1; cat $out/trace_bert.txt
timeout 120 python tools/attn_bench.py > $out/attn_bench.txt 2>&1; cat $out/attn_bench.txt
timeout 120 python tools/attn_bench.py > $out/attn_bench2.txt 2>&1; head -2 $out/attn_bench2.txt
for m in bert48; do
  timeout 600 python bench.py --model $m --steps 5 --warmup 3 --no-cpu > $out/${m}.json 2> $out/${m}.err
  echo "$m rc=$? $(python -c "import json; d=json.load(open('$out/${m}.json')); print(d['value'], d['e2e']['value'], d['clocks']['sm_mhz'], [ (k['kernel'], round(k.get('tflops',0))) for k in d['kernels'] if 'attention' in k['kernel']])" 2>&1 | tail -1)"
done
