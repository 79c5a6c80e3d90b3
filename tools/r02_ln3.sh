#!/bin/bash
# fused LayerNorm backward (rows + column partials) vs the three-launch form (DPL_LN_BWD_FUSED=0), same build
out=gpurun_out/r2ln3; mkdir -p $out
timeout 900 python -m pytest tests/test_elementwise_gpu.py tests/test_executor_gpu.py tests/test_baseline_shapes_gpu.py tests/test_lm_gpu.py -m gpu -q -x --timeout 300 --timeout-method thread -p no:cacheprovider -rf > $out/pytest.txt 2>&1
tail -1 $out/pytest.txt
DPL_LN_BWD_FUSED=0 timeout 300 python -m pytest tests/test_elementwise_gpu.py -m gpu -q -x -k layernorm -p no:cacheprovider > $out/pytest_unfused.txt 2>&1; tail -1 $out/pytest_unfused.txt
for v in 1 0 1 0; do
  echo "== fused=$v"; DPL_LN_BWD_FUSED=$v timeout 120 python tools/elementwise_graph_bench.py 2>&1 | grep layernorm_bwd
  DPL_LN_BWD_FUSED=$v timeout 120 python tools/elementwise_graph_bench.py --h 1600 --rows 1024 2>&1 | grep layernorm_bwd
done
for v in 1 0 1 0; do
  DPL_LN_BWD_FUSED=$v timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e > $out/bert_$v.json 2> $out/bert_$v.err
  python -c "import json; d=json.load(open('$out/bert_$v.json')); print('bert fused=$v', round(d['value'],2), d['clocks']['sm_mhz'], [(k['kernel'], round(k['seconds']*1e3,2)) for k in d['kernels'] if 'layernorm' in k['kernel']])"
done
for v in 1 0; do
  DPL_LN_BWD_FUSED=$v timeout 600 python bench.py --model gpt2-1.5b --steps 3 --warmup 3 --no-cpu --no-e2e > $out/gpt2_$v.json 2> $out/gpt2_$v.err
  python -c "import json; d=json.load(open('$out/gpt2_$v.json')); print('gpt2 fused=$v', round(d['value'],2), d['clocks']['sm_mhz'], [(k['kernel'], round(k['seconds']*1e3,2)) for k in d['kernels'] if 'layernorm' in k['kernel']])"
done
cmd="python tools/elementwise_graph_bench.py"
timeout 600 ncu --set full --clock-control none -k regex:'ln_bwd_fused|ln_param' -c 2 --csv --page raw --log-file $out/ln_fused_raw.csv $cmd > $out/ncu.log 2>&1; echo "ncu rc=$?"
