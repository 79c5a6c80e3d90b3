#!/bin/bash
# Late round-2 4-GPU confirmation: the full GPU suite on 4 GPUs and the N = 2 / 4 lines.
out=${OUT:-gpurun_out/r2f4e}; mkdir -p $out
timeout 1800 python -m pytest tests -m gpu -q --timeout 600 --timeout-method thread -p no:cacheprovider -rf > $out/pytest_4gpu.txt 2>&1
tail -2 $out/pytest_4gpu.txt
run() { # n tag args...
  local n=$1 tag=$2; shift 2
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29611 \
    bench.py --gpus $n --steps 5 --warmup 3 "$@" > $out/$tag.json 2> $out/$tag.err
  echo "$tag rc=$? $(python -c "import json; d=json.load(open('$out/$tag.json')); print(round(d['value'],2), round(d['e2e']['value'],2), d['clocks']['sm_mhz'], round(d['roofline']['frac'],4), d['config']['plan'], round(d.get('bubble') or 0,3), ((d.get('latency') or {}).get('planner') or {}).get('measured_over_planner_sim'))" 2>&1 | tail -1)"
}
run 2 bert_n2
run 4 bert_n4
run 4 gpt_n4 --model gpt2-1.5b
run 4 vgg_n4 --model vgg19
run 4 xlnet_n4 --model xlnet36 --plan planner
run 4 amoeba_n4 --model amoebanet36 --plan planner
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 \
  bench.py --impl reference --gpus 2 --steps 3 --warmup 3 > $out/ref_n2.json 2> $out/ref_n2.err; echo "ref n2 rc=$?"
