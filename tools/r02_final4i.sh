#!/bin/bash
# HEAD (late dW1 fork) on 4 GPUs: multi-GPU torchrun parity cases + BERT-48 N=2 / N=4
out=gpurun_out/r2f4i; mkdir -p $out
timeout 900 python -m pytest tests/test_executor_multigpu.py -m gpu -q --timeout 600 --timeout-method thread -p no:cacheprovider -rf > $out/pytest_mgpu.txt 2>&1; tail -1 $out/pytest_mgpu.txt
run() { local n=$1 tag=$2; shift 2
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29611 \
    bench.py --gpus $n --steps 5 --warmup 3 "$@" > $out/$tag.json 2> $out/$tag.err
  echo "$tag rc=$? $(python -c "import json; d=json.load(open('$out/$tag.json')); pl=d['latency'].get('planner') or {}; print(round(d['value'],2), round(d['e2e']['value'],2), d['clocks']['sm_mhz'], d['config']['plan'], round(d['bubble'],3), pl.get('measured_over_planner_sim'))" 2>&1 | tail -1)"
}
run 2 bert_n2
run 4 bert_n4
