#!/bin/bash
# 256 x 192 CTA-pair tiles: default (DPL_GEMM_BN192_COST=1.1) vs disabled (0), same build
out=gpurun_out/r2bn192; mkdir -p $out
timeout 900 python -m pytest tests/test_gemm_gpu.py -m gpu -q -x --timeout 300 --timeout-method thread -p no:cacheprovider -rf > $out/pytest.txt 2>&1
tail -1 $out/pytest.txt
for v in 1.1 0; do echo "== bn192 cost=$v"; DPL_GEMM_BN192_COST=$v timeout 300 python tools/gemm_graph_bench.py --T 1024 --H 1600 --F 6400 > $out/gg_gpt2_$v.txt 2>&1; python -c "
import json
for l in open('$out/gg_gpt2_$v.txt'):
    try: d=json.loads(l)
    except Exception: continue
    print(d.get('gemm'), d.get('ours_us'), d.get('cublas_us'), d.get('sum_us',''))"; done
for v in 1.1 0; do DPL_GEMM_BN192_COST=$v timeout 300 python tools/gemm_graph_bench.py --T 2048 > $out/gg_bert2048_$v.txt 2>&1; echo "bert2048 cost=$v $(tail -1 $out/gg_bert2048_$v.txt)"; done
for v in 1.1 0 1.1 0; do
  DPL_GEMM_BN192_COST=$v timeout 600 python bench.py --model gpt2-1.5b --steps 3 --warmup 3 --no-cpu --no-e2e > $out/gpt2_$v.json 2> $out/gpt2_$v.err
  python -c "import json; d=json.load(open('$out/gpt2_$v.json')); print('gpt2 cost=$v', round(d['value'],2), d['clocks']['sm_mhz'], round(d['roofline']['frac'],4))"
  DPL_GEMM_BN192_COST=$v timeout 600 python bench.py --global-batch 32 --steps 5 --warmup 3 --no-cpu --no-e2e --no-profile > $out/bert32_$v.json 2> $out/bert32_$v.err
  python -c "import json; d=json.load(open('$out/bert32_$v.json')); print('bert gbs32 cost=$v', round(d['value'],2), d['clocks']['sm_mhz'], round(d['roofline']['frac'],4))"
done
DPL_GEMM_BN192_COST=1.1 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e > $out/bert_1.1.json 2> $out/bert.err
python -c "import json; d=json.load(open('$out/bert_1.1.json')); print('bert n1 cost=1.1', round(d['value'],2), d['clocks']['sm_mhz'], round(d['roofline']['frac'],4))"
