#!/bin/bash
out=gpurun_out/r2pref; mkdir -p $out
timeout 600 python -m pytest tests/test_attention_gpu.py -m gpu -q -x --timeout 300 --timeout-method thread -p no:cacheprovider > $out/pytest.txt 2>&1; tail -1 $out/pytest.txt
timeout 100 python tools/attn_trace.py 8 512 16 0 --bwd 2>&1 | grep -E "S1 -> S2|S2 -> S3|lifetime|span"
timeout 100 python tools/attn_trace.py 8 512 16 0 2>&1 | grep -E "S1 -> S2|lifetime|span"
timeout 100 python tools/attn_bench.py 2>&1 | head -2
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu > $out/bert.json 2>/dev/null; python -c "import json; d=json.load(open('$out/bert.json')); print('bert', round(d['value'],2), d['clocks']['sm_mhz'])"
