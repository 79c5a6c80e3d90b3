#!/bin/bash
# Round-2 profiles (one GPU): launch list of a BERT-48 step, DRAM bytes of
# the HBM-bound kernels, and one full capture of the top GEMM (ffn1).
out=gpurun_out/r2ncu; mkdir -p $out
cmd="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-profile"
$cmd > $out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 3000 -c 1500 --csv --log-file $out/launches.csv $cmd > $out/ncu_launches.log 2>&1
echo "launches rc=$?"
$cmd > $out/plain2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed \
    --clock-control none -k regex:'layernorm|colsum|sgd|mse|attn|cross|embed' -s 200 -c 60 --csv --log-file $out/hbm_kernels.csv $cmd > $out/ncu_hbm.log 2>&1
echo "hbm rc=$?"
timeout 120 python tools/gemm_trace.py ffn1 > $out/plain3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gemm_bf16 -s 5 -c 1 -o $out/gemm_ffn1 python tools/gemm_trace.py ffn1 > $out/ncu_full.log 2>&1
echo "full rc=$?"
