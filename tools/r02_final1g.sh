#!/bin/bash
# Closing 1-GPU confirmation of HEAD + the planner's N = 2 / 4 / 8 choices from this GPU's profiles
out=gpurun_out/r2f1g; mkdir -p $out
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 --timeout-method thread -p no:cacheprovider -rf > $out/pytest_1gpu.txt 2>&1
tail -1 $out/pytest_1gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke rc=$? $(tail -1 $out/smoke.log)"
timeout 900 python bench.py > $out/bert_n1.json 2> $out/bert_n1.err; echo "bert rc=$? $(python -c "import json; d=json.load(open('$out/bert_n1.json')); print(round(d['value'],2), round(d['e2e']['value'],2), d['clocks']['sm_mhz'], round(d['roofline']['frac'],4))" 2>&1 | tail -1)"
timeout 900 python bench.py --model gpt2-1.5b --steps 5 --warmup 3 > $out/gpt2_n1.json 2> $out/gpt2_n1.err; echo "gpt2 rc=$? $(python -c "import json; d=json.load(open('$out/gpt2_n1.json')); print(round(d['value'],2), round(d['e2e']['value'],2), d['clocks']['sm_mhz'], round(d['roofline']['frac'],4))" 2>&1 | tail -1)"
timeout 900 python tools/plan8.py > $out/plan8_bert.jsonl 2> $out/plan8_bert.err; echo "plan8 bert rc=$?"; cat $out/plan8_bert.jsonl
timeout 900 python tools/plan8.py --model xlnet36 > $out/plan8_xlnet.jsonl 2> $out/plan8_xlnet.err; echo "plan8 xlnet rc=$?"; cat $out/plan8_xlnet.jsonl
