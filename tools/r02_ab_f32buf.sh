#!/bin/bash
# fp32 reduce-add GEMM outputs (weight gradients): one staging buffer per
# warp + a sixth ring stage (DPL_GEMM_F32_OUT_BUFS=1) vs double-buffered (default)
out=gpurun_out/r2abf32; mkdir -p $out
DPL_GEMM_F32_OUT_BUFS=1 timeout 900 python -m pytest tests/test_gemm_gpu.py tests/test_vgg_gpu.py tests/test_executor_gpu.py -m gpu -q -x --timeout 300 --timeout-method thread -p no:cacheprovider > $out/pytest.txt 2>&1; tail -1 $out/pytest.txt
for r in 1 2; do for v in 2 1; do
  export DPL_GEMM_F32_OUT_BUFS=$v
  timeout 200 python tools/gemm_graph_bench.py > $out/gg_${v}_$r.txt 2>&1; echo "bufs=$v"; python tools/gg_summary.py $out/gg_${v}_$r.txt | grep "wgrad\|sum"
  for m in bert48 gpt2-1.5b vgg19; do
    timeout 600 python bench.py --model $m --steps 5 --warmup 3 --no-cpu > $out/${m}_${v}_$r.json 2>/dev/null
    echo "  $m bufs=$v $(python -c "import json; d=json.load(open('$out/${m}_${v}_$r.json')); print(round(d['value'],2), d['clocks']['sm_mhz'])" 2>&1 | tail -1)"
  done
done; done
