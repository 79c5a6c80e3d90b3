#!/bin/bash
# dWo forked after the attention backward (DPL_WO_LATE=1) vs before the O dgrad (default)
out=gpurun_out/r2wolate; mkdir -p $out
DPL_WO_LATE=1 timeout 600 python -m pytest tests/test_executor_gpu.py -m gpu -q -x --timeout 300 --timeout-method thread -p no:cacheprovider > $out/pytest.txt 2>&1; tail -1 $out/pytest.txt
for rep in 1 2; do for v in 1 0; do
  DPL_WO_LATE=$v timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --no-profile > $out/bert_${v}_$rep.json 2> $out/bert_${v}_$rep.err
  python -c "import json; d=json.load(open('$out/bert_${v}_$rep.json')); print('bert wo_late=$v', round(d['value'],2), d['clocks']['sm_mhz'], [(k['kernel'], round(k['seconds']*1e3,1)) for k in d['kernels'][:5]])"
done; done
