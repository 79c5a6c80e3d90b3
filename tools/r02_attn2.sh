#!/bin/bash
# mbarrier waits with a suspend-time hint + attention forward S_{j+1}-before-PV_j
# ordering / double-buffered K: GPU tests, N=1 bench lines, ncu of both
# attention kernels and the top GEMM at BERT-48's shape.
out=gpurun_out/r2attn2; mkdir -p $out
timeout 1200 python -m pytest tests -m gpu -q --timeout 400 --timeout-method thread -p no:cacheprovider -rf -x > $out/pytest.txt 2>&1
tail -2 $out/pytest.txt
for m in bert48 gpt2-1.5b vgg19; do
  timeout 600 python bench.py --model $m --steps 5 --warmup 3 --no-cpu > $out/${m}.json 2> $out/${m}.err
  echo "$m rc=$? $(python -c "import json; d=json.load(open('$out/${m}.json')); print(d['value'], d['e2e']['value'], d['clocks']['sm_mhz'], d['roofline']['achieved'])" 2>&1 | tail -1)"
done
cmd="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-profile"
$cmd > $out/plain.log 2>&1 && {
timeout 600 ncu --set full --import-source on --clock-control none -k regex:'attn_fwd_kernel' --launch-skip 4 -c 1 -o $out/attn_fwd $cmd > $out/ncu_fwd.log 2>&1; echo "ncu fwd rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:'attn_bwd_kernel' --launch-skip 4 -c 1 -o $out/attn_bwd $cmd > $out/ncu_bwd.log 2>&1; echo "ncu bwd rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file $out/launches.csv $cmd > $out/ncu_launches.log 2>&1; echo "ncu launches rc=$?"
}
