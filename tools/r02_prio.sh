#!/bin/bash
# stream priorities (compute high / wgrad low) and side-stream GEMM grid caps
out=gpurun_out/r2prio; mkdir -p $out
run() { # tag env... model
  local tag=$1 m=$2; shift 2
  env "$@" timeout 600 python bench.py --model $m --steps 5 --warmup 3 --no-cpu > $out/${tag}_${m}.json 2> $out/${tag}_${m}.err
  echo "$tag $m $(python -c "import json; d=json.load(open('$out/${tag}_${m}.json')); print(round(d['value'],2), d['clocks']['sm_mhz'])" 2>&1 | tail -1)"
}
for m in bert48 gpt2-1.5b; do
  run noprio $m DPL_STREAM_PRIO=0
  run prio $m DPL_STREAM_PRIO=1
  run cap96 $m DPL_WGRAD_CTAS=96
  run cap64 $m DPL_WGRAD_CTAS=64
  run cap32 $m DPL_WGRAD_CTAS=32
  run noprio2 $m DPL_STREAM_PRIO=0
  run prio2 $m DPL_STREAM_PRIO=1
done
run prio vgg19 DPL_STREAM_PRIO=1
run noprio vgg19 DPL_STREAM_PRIO=0
