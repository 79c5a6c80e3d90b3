#!/bin/bash
# split-K for small bf16 GEMMs, re-measured with the weight-gradient side stream on
out=gpurun_out/r2absplit; mkdir -p $out
for r in 1 2; do for v in 0 1; do
  DPL_GEMM_SPLIT_BF16=$v timeout 600 python bench.py --model gpt2-1.5b --steps 5 --warmup 3 --no-cpu > $out/gpt_s${v}_$r.json 2>/dev/null
  echo "gpt split=$v $(python -c "import json; d=json.load(open('$out/gpt_s${v}_$r.json')); print(round(d['value'],2), d['clocks']['sm_mhz'])")"
  DPL_GEMM_SPLIT_BF16=$v timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --global-batch 16 --no-e2e > $out/bert16_s${v}_$r.json 2>/dev/null
  echo "bert gbs16 split=$v $(python -c "import json; d=json.load(open('$out/bert16_s${v}_$r.json')); print(round(d['value'],2), d['clocks']['sm_mhz'])")"
done; done
