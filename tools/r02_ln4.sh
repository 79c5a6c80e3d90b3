#!/bin/bash
# fused LayerNorm backward: 2 x 256-thread blocks per SM (default) vs 1 x 512 vs the three-launch form
out=gpurun_out/r2ln4; mkdir -p $out
timeout 900 python -m pytest tests/test_elementwise_gpu.py tests/test_executor_gpu.py -m gpu -q -x --timeout 300 --timeout-method thread -p no:cacheprovider -rf > $out/pytest.txt 2>&1
tail -1 $out/pytest.txt
DPL_LN_FUSED_BPS=1 timeout 300 python -m pytest tests/test_elementwise_gpu.py -m gpu -q -x -k layernorm -p no:cacheprovider > $out/pytest_bps1.txt 2>&1; tail -1 $out/pytest_bps1.txt
for v in "1 2" "1 1" "0 2" "1 2" "1 1" "0 2"; do
  set -- $v
  echo "== fused=$1 bps=$2"; DPL_LN_BWD_FUSED=$1 DPL_LN_FUSED_BPS=$2 timeout 120 python tools/elementwise_graph_bench.py 2>&1 | grep layernorm_bwd
  DPL_LN_BWD_FUSED=$1 DPL_LN_FUSED_BPS=$2 timeout 120 python tools/elementwise_graph_bench.py --h 1600 --rows 1024 2>&1 | grep layernorm_bwd
done
for v in "1 2" "1 1" "0 2" "1 2" "1 1" "0 2"; do
  set -- $v
  DPL_LN_BWD_FUSED=$1 DPL_LN_FUSED_BPS=$2 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e > $out/bert_$1_$2.json 2> $out/bert_$1_$2.err
  python -c "import json; d=json.load(open('$out/bert_$1_$2.json')); print('bert fused=$1 bps=$2', round(d['value'],2), d['clocks']['sm_mhz'], [(k['kernel'], round(k['seconds']*1e3,2)) for k in d['kernels'] if 'layernorm' in k['kernel']])"
done
for v in "1 2" "0 2"; do
  set -- $v
  DPL_LN_BWD_FUSED=$1 timeout 600 python bench.py --model gpt2-1.5b --steps 3 --warmup 3 --no-cpu --no-e2e > $out/gpt2_$1.json 2> $out/gpt2_$1.err
  python -c "import json; d=json.load(open('$out/gpt2_$1.json')); print('gpt2 fused=$1', round(d['value'],2), d['clocks']['sm_mhz'], [(k['kernel'], round(k['seconds']*1e3,2)) for k in d['kernels'] if 'layernorm' in k['kernel']])"
done
timeout 600 ncu --set full --clock-control none -k regex:'ln_bwd_fused|ln_param' -c 2 --csv --page raw --log-file $out/ln_fused_raw.csv python tools/elementwise_graph_bench.py > $out/ncu.log 2>&1; echo "ncu rc=$?"
