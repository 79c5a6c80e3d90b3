#!/bin/bash
# Round-2 multi-GPU confirmation (run under gpurun --gpus 4): the multi-GPU
# parity suite (peer-memory AllReduce by default), then bench lines at N = 2
# and 4 for C2 (planner plan, GBS 64) with both AllReduce implementations,
# and the C5 XLNet-36 stand-in on the planner's plans.
out=gpurun_out/r2mg; mkdir -p $out
nvidia-smi topo -m > $out/topo.txt 2>&1
if [ "${SKIP_TESTS:-0}" != 1 ]; then
  timeout 1800 python -m pytest tests -m gpu -q --timeout 600 --timeout-method thread -p no:cacheprovider -rf > $out/pytest_mgpu.txt 2>&1
  tail -5 $out/pytest_mgpu.txt
fi
run() { # n tag args...
  local n=$1 tag=$2; shift 2
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29611 \
    bench.py --gpus $n --steps 5 --warmup 3 "$@" > $out/$tag.json 2> $out/$tag.err; echo "$tag rc=$?"
}
run 2 bert_n2
run 4 bert_n4
DPL_ALLREDUCE=nccl run 4 bert_n4_nccl
run 4 bert_n4_timeline --timeline-out $out/timelines
run 4 xlnet_n4 --model xlnet36 --plan planner
run 2 xlnet_n2 --model xlnet36 --plan planner
timeout 900 python bench.py --model xlnet36 --plan planner --no-cpu > $out/xlnet_n1.json 2> $out/xlnet_n1.err; echo "xlnet_n1 rc=$?"
