#!/bin/bash
# XLNet-36 / AmoebaNet-36 stand-ins at N=4 with the multi-start planner fixed point
out=gpurun_out/r2x4; mkdir -p $out
run() { local n=$1 tag=$2; shift 2
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29613 \
    bench.py --gpus $n --steps 5 --warmup 3 "$@" > $out/$tag.json 2> $out/$tag.err; echo "$tag rc=$?"; }
run 4 xlnet_n4 --model xlnet36 --plan planner
run 4 amoeba_n4 --model amoebanet36 --plan planner
run 2 xlnet_n2 --model xlnet36 --plan planner
run 2 amoeba_n2 --model amoebanet36 --plan planner
run 2 vgg_n2 --model vgg19
