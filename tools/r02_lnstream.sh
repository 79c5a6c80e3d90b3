#!/bin/bash
# LayerNorm-backward parameter passes on their own stream: GPU tests + A/B
out=gpurun_out/r2lns; mkdir -p $out
timeout 1200 python -m pytest tests/test_executor_gpu.py tests/test_lm_gpu.py tests/test_baseline_shapes_gpu.py tests/test_executor_api_gpu.py tests/test_elementwise_gpu.py -m gpu -q -x --timeout 400 --timeout-method thread -p no:cacheprovider -rf > $out/pytest.txt 2>&1
tail -1 $out/pytest.txt
for r in 1 2; do for v in 0 1; do
  for m in bert48 gpt2-1.5b; do
    DPL_LN_STREAM=$v timeout 600 python bench.py --model $m --steps 5 --warmup 3 --no-cpu > $out/${m}_ln${v}_$r.json 2>/dev/null
    echo "$m ln_stream=$v $(python -c "import json; d=json.load(open('$out/${m}_ln${v}_$r.json')); print(round(d['value'],2), d['clocks']['sm_mhz'])" 2>&1 | tail -1)"
  done
done; done
