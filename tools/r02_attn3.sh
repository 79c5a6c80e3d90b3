#!/bin/bash
# two-threads-per-row attention forward + backward MMA reorder: attention /
# LM / baseline-shape tests, trace, kernel bench, BERT / GPT-2 N=1 lines.
out=gpurun_out/r2attn3; mkdir -p $out
timeout 600 python -m pytest tests/test_attention_gpu.py tests/test_lm_gpu.py -m gpu -q -x --timeout 300 --timeout-method thread -p no:cacheprovider -rf > $out/pytest_attn.txt 2>&1
tail -2 $out/pytest_attn.txt
timeout 120 python tools/attn_trace.py 8 512 16 0 > $out/trace_bert.txt 2>&1; cat $out/trace_bert.txt
timeout 120 python tools/attn_trace.py 1 1024 25 1 > $out/trace_gpt.txt 2>&1; tail -4 $out/trace_gpt.txt
timeout 120 python tools/attn_bench.py > $out/attn_bench.txt 2>&1; head -2 $out/attn_bench.txt
timeout 900 python -m pytest tests -m gpu -q -x --timeout 400 --timeout-method thread -p no:cacheprovider -rf > $out/pytest.txt 2>&1
tail -2 $out/pytest.txt
for m in bert48 gpt2-1.5b; do
  timeout 600 python bench.py --model $m --steps 5 --warmup 3 --no-cpu > $out/${m}.json 2> $out/${m}.err
  echo "$m rc=$? $(python -c "import json; d=json.load(open('$out/${m}.json')); print(d['value'], d['e2e']['value'], d['clocks']['sm_mhz'], [ (k['kernel'], round(k.get('tflops',0))) for k in d['kernels'] if 'attention' in k['kernel']])" 2>&1 | tail -1)"
done
