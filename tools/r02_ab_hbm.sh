#!/bin/bash
# A/B: LayerNorm-backward rows with the residual gradient fetched by cp.async
# alongside x / dy, and colsum at four blocks per SM (new) vs before (old)
out=gpurun_out/r2abhbm; mkdir -p $out
cp abtmp/libdapple_new.so paper_2007_01045_b200/libdapple.so
timeout 900 python -m pytest tests/test_elementwise_gpu.py tests/test_executor_gpu.py tests/test_lm_gpu.py tests/test_baseline_shapes_gpu.py -m gpu -q -x --timeout 300 --timeout-method thread -p no:cacheprovider > $out/pytest.txt 2>&1; tail -1 $out/pytest.txt
for r in 1 2; do for v in old new; do
  cp abtmp/libdapple_$v.so paper_2007_01045_b200/libdapple.so
  echo "$v: $(timeout 100 python tools/attn_bench.py 2>&1 | tail -5 | tr '\n' ';')"
  for m in bert48 gpt2-1.5b; do
    timeout 600 python bench.py --model $m --steps 5 --warmup 3 --no-cpu > $out/${v}_${m}_$r.json 2>/dev/null
    echo "  $v $m $(python -c "import json; d=json.load(open('$out/${v}_${m}_$r.json')); print(round(d['value'],2), d['clocks']['sm_mhz'])" 2>&1 | tail -1)"
  done
done; done
cp abtmp/libdapple_new.so paper_2007_01045_b200/libdapple.so
