#!/bin/bash
# W1 weight gradient forked after the LN2 backward (DPL_WGRAD_LATE=1) vs before (default), same build
out=gpurun_out/r2wlate; mkdir -p $out
DPL_WGRAD_LATE=1 timeout 600 python -m pytest tests/test_executor_gpu.py tests/test_baseline_shapes_gpu.py -m gpu -q -x --timeout 300 --timeout-method thread -p no:cacheprovider > $out/pytest.txt 2>&1; tail -1 $out/pytest.txt
for rep in 1 2; do for v in 1 0; do
  DPL_WGRAD_LATE=$v timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --no-profile > $out/bert_${v}_$rep.json 2> $out/bert_${v}_$rep.err
  python -c "import json; d=json.load(open('$out/bert_${v}_$rep.json')); print('bert late=$v', round(d['value'],2), d['clocks']['sm_mhz'], round(d['roofline']['frac'],4), [(k['kernel'], round(k['seconds']*1e3,1)) for k in d['kernels'][:5]])"
  DPL_WGRAD_LATE=$v timeout 600 python bench.py --model gpt2-1.5b --steps 3 --warmup 3 --no-cpu --no-e2e --no-profile > $out/gpt2_${v}_$rep.json 2> $out/gpt2_${v}_$rep.err
  python -c "import json; d=json.load(open('$out/gpt2_${v}_$rep.json')); print('gpt2 late=$v', round(d['value'],2), d['clocks']['sm_mhz'])"
done; done
