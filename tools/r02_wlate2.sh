#!/bin/bash
# default (late fork for full-machine side grids) confirmation
out=gpurun_out/r2wlate2; mkdir -p $out
timeout 900 python -m pytest tests/test_executor_gpu.py tests/test_baseline_shapes_gpu.py tests/test_local_ranks_gpu.py tests/test_lm_gpu.py -m gpu -q -x --timeout 300 --timeout-method thread -p no:cacheprovider > $out/pytest.txt 2>&1; tail -1 $out/pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke rc=$? $(tail -1 $out/smoke.log)"
timeout 900 python bench.py > $out/bert_n1.json 2> $out/bert_n1.err; echo "bert rc=$? $(python -c "import json; d=json.load(open('$out/bert_n1.json')); print(round(d['value'],2), round(d['e2e']['value'],2), d['clocks']['sm_mhz'], round(d['roofline']['frac'],4))" 2>&1 | tail -1)"
timeout 600 python bench.py --model gpt2-1.5b --steps 3 --warmup 3 --no-cpu > $out/gpt2_n1.json 2> $out/gpt2_n1.err; echo "gpt2 rc=$? $(python -c "import json; d=json.load(open('$out/gpt2_n1.json')); print(round(d['value'],2), d['clocks']['sm_mhz'])" 2>&1 | tail -1)"
timeout 600 python bench.py --model xlnet36 --steps 3 --warmup 3 --no-cpu > $out/xlnet_n1.json 2> $out/xlnet_n1.err; echo "xlnet rc=$? $(python -c "import json; d=json.load(open('$out/xlnet_n1.json')); print(round(d['value'],2), d['clocks']['sm_mhz'])" 2>&1 | tail -1)"
