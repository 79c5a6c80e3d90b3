#!/bin/bash
# Final 4-GPU confirmation of the round-2 tree.
out=${OUT:-gpurun_out/r2f6}; mkdir -p $out
timeout 1800 python -m pytest tests -m gpu -q --timeout 600 --timeout-method thread -p no:cacheprovider -rf > $out/pytest_4gpu.txt 2>&1
tail -3 $out/pytest_4gpu.txt
run() { # n tag args...
  local n=$1 tag=$2; shift 2
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29611 \
    bench.py --gpus $n --steps 5 --warmup 3 "$@" > $out/$tag.json 2> $out/$tag.err; echo "$tag rc=$?"
}
run 4 bert_n4 --timeline-out $out/timelines
run 2 bert_n2
run 4 gpt_n4 --model gpt2-1.5b
run 4 vgg_n4 --model vgg19
DPL_ALLREDUCE=nccl run 4 bert_n4_nccl
run 4 xlnet_n4 --model xlnet36 --plan planner
run 4 amoeba_n4 --model amoebanet36 --plan planner
