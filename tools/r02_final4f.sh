#!/bin/bash
# planner fixed point with the top-k runners-up priced: BERT-48 N=2 / 4 (default plan path), C5 stand-ins at N=4
out=${OUT:-gpurun_out/r2f4f}; mkdir -p $out
run() { # n tag args...
  local n=$1 tag=$2; shift 2
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29611 \
    bench.py --gpus $n --steps 5 --warmup 3 "$@" > $out/$tag.json 2> $out/$tag.err
  echo "$tag rc=$? $(python -c "import json; d=json.load(open('$out/$tag.json')); pl=d['latency'].get('planner') or {}; print(round(d['value'],2), round(d['e2e']['value'],2), d['clocks']['sm_mhz'], d['config']['plan'], round(d['bubble'],3), pl.get('measured_over_planner_sim'), pl.get('candidates'))" 2>&1 | tail -1)"
}
run 2 bert_n2
run 4 bert_n4
run 4 xlnet_n4 --model xlnet36 --plan planner
run 2 xlnet_n2 --model xlnet36 --plan planner
run 4 amoeba_n4 --model amoebanet36 --plan planner
