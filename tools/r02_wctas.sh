#!/bin/bash
# side-stream (weight-gradient) GEMM grid cap at BERT-48's 4096-row slices: DPL_WGRAD_CTAS 0 (default: full machine) / 96 / 112 / 128
out=gpurun_out/r2wctas; mkdir -p $out
for rep in 1 2; do for v in 0 96 112 128; do
  DPL_WGRAD_CTAS=$v timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --no-profile > $out/bert_${v}_$rep.json 2> $out/bert_${v}_$rep.err
  python -c "import json; d=json.load(open('$out/bert_${v}_$rep.json')); print('bert ctas=$v', round(d['value'],2), d['clocks']['sm_mhz'], round(d['roofline']['frac'],4), [(k['kernel'], round(k['seconds']*1e3,1)) for k in d['kernels'][:5]])"
done; done
