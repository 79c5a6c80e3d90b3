#!/bin/bash
# split-K threshold: K blocks >= 16 (all small-slice N=1600 GEMMs) vs >= 48 (only K >= 3072) vs off
out=gpurun_out/r2abskb; mkdir -p $out
for r in 1 2; do for v in 16 48 off; do
  if [ $v = off ]; then env="DPL_GEMM_SPLIT_BF16=0"; else env="DPL_GEMM_SPLIT_MIN_KB=$v"; fi
  env $env timeout 600 python bench.py --model gpt2-1.5b --steps 5 --warmup 3 --no-cpu > $out/gpt_${v}_$r.json 2>/dev/null
  echo "gpt $v $(python -c "import json; d=json.load(open('$out/gpt_${v}_$r.json')); print(round(d['value'],2), d['clocks']['sm_mhz'])" 2>&1 | tail -1)"
done; done
