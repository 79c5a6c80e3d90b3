#!/bin/bash
# elected MMA issue from a converged warp (attention + GEMM): tests, traces,
# kernel bench, N=1 lines
out=gpurun_out/r2elect; mkdir -p $out
timeout 900 python -m pytest tests/test_attention_gpu.py tests/test_gemm_gpu.py tests/test_vgg_gpu.py -m gpu -q -x --timeout 300 --timeout-method thread -p no:cacheprovider -rf > $out/pytest.txt 2>&1
tail -1 $out/pytest.txt
timeout 100 python tools/attn_trace.py 8 512 16 0 2>&1 | grep -E "S1 -> S2|lifetime|span"
timeout 100 python tools/attn_trace.py 8 512 16 0 --bwd 2>&1 | grep -E "S1 -> S2|S2 -> S3|lifetime|span"
timeout 100 python tools/attn_bench.py 2>&1 | head -2
for m in bert48 gpt2-1.5b vgg19; do
  timeout 600 python bench.py --model $m --steps 5 --warmup 3 --no-cpu > $out/${m}.json 2> $out/${m}.err
  echo "$m rc=$? $(python -c "import json; d=json.load(open('$out/${m}.json')); print(round(d['value'],2), round(d['e2e']['value'],2), d['clocks']['sm_mhz'], round(d['roofline']['achieved']), [ (k['kernel'], round(k.get('tflops',0))) for k in d['kernels'] if 'attention' in k['kernel']])" 2>&1 | tail -1)"
done
