#!/bin/bash
# HEAD 1-GPU evidence: GPU suite, smoke, N=1 lines of every workload (+ reference arm), BERT-48 launch list
out=gpurun_out/r2f1h; mkdir -p $out
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 --timeout-method thread -p no:cacheprovider -rf > $out/pytest_1gpu.txt 2>&1
tail -1 $out/pytest_1gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke rc=$? $(tail -1 $out/smoke.log)"
timeout 900 python bench.py > $out/bert_n1.json 2> $out/bert_n1.err; echo "bert rc=$? $(python -c "import json; d=json.load(open('$out/bert_n1.json')); print(round(d['value'],2), round(d['e2e']['value'],2), d['clocks']['sm_mhz'], d['clocks']['reasons'], round(d['roofline']['frac'],4))" 2>&1 | tail -1)"
timeout 900 python bench.py --impl reference > $out/ref_n1.json 2> $out/ref_n1.err; echo "ref rc=$?"
for m in gpt2-1.5b vgg19 xlnet36 amoebanet36; do
  timeout 900 python bench.py --model $m --steps 5 --warmup 3 > $out/${m}_n1.json 2> $out/${m}_n1.err
  echo "$m rc=$? $(python -c "import json; d=json.load(open('$out/${m}_n1.json')); print(round(d['value'],2), round(d['e2e']['value'],2), d['clocks']['sm_mhz'], round(d['roofline']['frac'],4))" 2>&1 | tail -1)"
done
cmd="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-profile"
$cmd > $out/plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --launch-skip 600 --csv --log-file $out/launches.csv $cmd > $out/ncu_launches.log 2>&1; echo "launches rc=$?"
python tools/launch_shares.py $out/launches.csv > $out/launch_shares.txt 2>&1; head -12 $out/launch_shares.txt
