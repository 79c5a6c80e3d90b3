#!/bin/bash
# ncu --set full of the final GEMM kernel at the three heaviest BERT-48 shapes
out=gpurun_out/r2gncu; mkdir -p $out
for g in ffn1 o ffn2; do
  timeout 120 python tools/gemm_one.py $g > $out/plain_$g.log 2>&1 && \
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm_bf16 --launch-skip 3 -c 1 -o $out/gemm_$g python tools/gemm_one.py $g > $out/ncu_$g.log 2>&1
  echo "$g rc=$?"
done
