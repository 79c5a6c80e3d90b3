#!/bin/bash
# fp32-accumulate split-K at any split count (DPL_GEMM_SPLIT_ANY=1, default) vs powers of two
out=gpurun_out/r2splitany; mkdir -p $out
timeout 900 python -m pytest tests/test_gemm_gpu.py -m gpu -q -x --timeout 300 --timeout-method thread -p no:cacheprovider -rf > $out/pytest.txt 2>&1
tail -1 $out/pytest.txt
for v in 1 0; do DPL_GEMM_SPLIT_ANY=$v timeout 300 python tools/gemm_graph_bench.py > $out/gg_$v.txt 2>&1; echo "== any=$v"; grep -h wgrad $out/gg_$v.txt | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['gemm'], d['ours_us'], d['cublas_us'])"; tail -1 $out/gg_$v.txt; done
for v in 1 0 1 0; do
  DPL_GEMM_SPLIT_ANY=$v timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e > $out/bert_$v.json 2> $out/bert_$v.err
  python -c "import json; d=json.load(open('$out/bert_$v.json')); print('bert any=$v', round(d['value'],2), d['clocks']['sm_mhz'], round(d['roofline']['frac'],4))"
done
for m in vgg19 amoebanet36; do for v in 1 0; do
  DPL_GEMM_SPLIT_ANY=$v timeout 600 python bench.py --model $m --steps 5 --warmup 3 --no-cpu --no-e2e > $out/${m}_$v.json 2> $out/${m}_$v.err
  python -c "import json; d=json.load(open('$out/${m}_$v.json')); print('$m any=$v', round(d['value'],2), d['clocks']['sm_mhz'], round(d['roofline']['frac'],4))"
done; done
