#!/bin/bash
# Final 4-GPU lines of the round-2 tree (GPU suite ran on the previous
# 4-GPU call; this one refreshes the bench lines after the last GEMM changes)
out=${OUT:-gpurun_out/r2f7}; mkdir -p $out
run() { # n tag args...
  local n=$1 tag=$2; shift 2
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29621 \
    bench.py --gpus $n --steps 5 --warmup 3 "$@" > $out/$tag.json 2> $out/$tag.err; echo "$tag rc=$?"
}
run 4 bert_n4 --timeline-out $out/timelines
run 2 bert_n2
run 4 gpt_n4 --model gpt2-1.5b
run 4 vgg_n4 --model vgg19
run 2 vgg_n2 --model vgg19
run 4 xlnet_n4 --model xlnet36 --plan planner
run 4 amoeba_n4 --model amoebanet36 --plan planner
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29622 \
  bench.py --impl reference --gpus 2 --steps 2 --warmup 1 > $out/ref_n2.json 2> $out/ref_n2.err; echo "ref_n2 rc=$?"
