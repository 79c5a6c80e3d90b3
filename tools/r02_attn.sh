#!/bin/bash
# Side-stream weight gradients for every layer kind (A/B), the GPU tests they
# touch, and one ncu --set full capture of each attention kernel at BERT-48's
# shape (s 512, 16 heads, 8-sample micro-batch).
out=gpurun_out/r2attn; mkdir -p $out
timeout 900 python -m pytest tests/test_vgg_gpu.py tests/test_executor_gpu.py tests/test_baseline_shapes_gpu.py tests/test_lm_gpu.py \
  -m gpu -q --timeout 400 --timeout-method thread -p no:cacheprovider -rf > $out/pytest.txt 2>&1
tail -2 $out/pytest.txt
for round in 1 2; do
  for ws in 0 1; do
    for m in vgg19 gpt2-1.5b bert48; do
      DPL_WGRAD_STREAM=$ws timeout 600 python bench.py --model $m --steps 5 --warmup 3 --no-cpu > $out/${m}_ws${ws}_r${round}.json 2> $out/${m}_ws${ws}_r${round}.err
      echo "$m ws=$ws r$round rc=$? $(python -c "import json,sys; d=json.load(open('$out/${m}_ws${ws}_r${round}.json')); print(d['value'], d['e2e']['value'], d['clocks']['sm_mhz'])" 2>&1 | tail -1)"
    done
  done
done
cmd="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-profile"
$cmd > $out/plain.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:'attn_fwd_kernel|attn_bwd_kernel' --launch-skip 4 -c 2 -o $out/attn $cmd > $out/ncu.log 2>&1; echo "ncu rc=$?"
