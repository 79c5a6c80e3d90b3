#!/bin/bash
# GEMM split tail (last wave as 256x128 halves) A/B: DPL_GEMM_SPLIT_TAIL=1 (default) vs 0, same build
out=gpurun_out/r2tail; mkdir -p $out
timeout 900 python -m pytest tests/test_gemm_gpu.py -m gpu -q -x --timeout 300 --timeout-method thread -p no:cacheprovider -rf > $out/pytest.txt 2>&1
tail -1 $out/pytest.txt
for v in 1 0 1 0; do
  echo "== tail=$v"; DPL_GEMM_SPLIT_TAIL=$v timeout 300 python tools/gemm_graph_bench.py > $out/gg_$v.txt 2>&1; tail -16 $out/gg_$v.txt
done
for v in 1 0 1 0; do
  DPL_GEMM_SPLIT_TAIL=$v timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e > $out/bert_$v.json 2> $out/bert_$v.err
  python -c "import json; d=json.load(open('$out/bert_$v.json')); print('bert tail=$v', round(d['value'],2), d['clocks']['sm_mhz'], round(d['roofline']['frac'],4))"
done
for v in 1 0; do
  DPL_GEMM_SPLIT_TAIL=$v timeout 600 python bench.py --model gpt2-1.5b --steps 3 --warmup 3 --no-cpu --no-e2e > $out/gpt2_$v.json 2> $out/gpt2_$v.err
  python -c "import json; d=json.load(open('$out/gpt2_$v.json')); print('gpt2 tail=$v', round(d['value'],2), d['clocks']['sm_mhz'], round(d['roofline']['frac'],4))"
done
