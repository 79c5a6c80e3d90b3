#!/bin/bash
out=gpurun_out/r2attn5; mkdir -p $out
timeout 600 python -m pytest tests/test_attention_gpu.py -m gpu -q -x --timeout 300 --timeout-method thread -p no:cacheprovider -rf > $out/pytest_attn.txt 2>&1
tail -1 $out/pytest_attn.txt
timeout 120 python tools/attn_trace.py 8 512 16 0 --bwd > $out/trace_bwd.txt 2>&1; cat $out/trace_bwd.txt
timeout 120 python tools/attn_trace.py 1 1024 25 1 --bwd > $out/trace_bwd_gpt.txt 2>&1; tail -5 $out/trace_bwd_gpt.txt
timeout 120 python tools/attn_bench.py > $out/attn_bench.txt 2>&1; head -2 $out/attn_bench.txt
