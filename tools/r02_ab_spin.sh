#!/bin/bash
# A/B: mbarrier waits with the suspend-time hint (default build) vs plain spinning
out=gpurun_out/r2spin; mkdir -p $out
for v in hint spin hint spin; do
  if [ $v = spin ]; then cp abtmp/libdapple_spin.so paper_2007_01045_b200/libdapple.so; else cp abtmp/libdapple_hint.so paper_2007_01045_b200/libdapple.so; fi
  echo "== $v"
  timeout 100 python tools/attn_trace.py 8 512 16 0 --bwd 2>&1 | grep -E "S1 -> S2|S2 -> S3|lifetime|span"
  timeout 100 python tools/attn_trace.py 8 512 16 0 2>&1 | grep -E "S1 -> S2|lifetime|span"
  timeout 100 python tools/attn_bench.py 2>&1 | head -1
done
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu > $out/bert_spin.json 2>/dev/null; python -c "import json; d=json.load(open('$out/bert_spin.json')); print('spin bert', d['value'], d['clocks']['sm_mhz'])"
cp abtmp/libdapple_hint.so paper_2007_01045_b200/libdapple.so
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu > $out/bert_hint.json 2>/dev/null; python -c "import json; d=json.load(open('$out/bert_hint.json')); print('hint bert', d['value'], d['clocks']['sm_mhz'])"
