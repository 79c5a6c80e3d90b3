#!/bin/bash
# DRAM bytes of the remaining HBM-bound kernels (LayerNorm forward / column
# pass / parameter reduce, MSE, SGD on BERT-48; cross-entropy and embedding
# on GPT-2 1.5B).
out=gpurun_out/r2ncu2; mkdir -p $out
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed"
cmd="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-profile"
$cmd > $out/plain.log 2>&1 && \
ncu --metrics $M --clock-control none -k regex:'layernorm_fwd|ln_bwd_cols|ln_param_reduce|mse|colsum' -c 40 --csv --log-file $out/ln.csv $cmd > $out/ncu_ln.log 2>&1; echo "ln rc=$?"
ncu --metrics $M --clock-control none -k regex:'sgd' -c 6 --csv --log-file $out/sgd.csv $cmd > $out/ncu_sgd.log 2>&1; echo "sgd rc=$?"
g="python bench.py --model gpt2-1.5b --steps 1 --warmup 1 --no-e2e --no-cpu --no-profile"
$g > $out/plain_gpt.log 2>&1 && \
ncu --metrics $M --clock-control none -k regex:'ce_kernel|embed' -c 6 --csv --log-file $out/lm.csv $g > $out/ncu_lm.log 2>&1; echo "lm rc=$?"
