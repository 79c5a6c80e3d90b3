#!/bin/bash
# early programmatic-launch triggers in the elementwise / attention-helper kernels: new lib vs ab/libdapple_old.so
out=gpurun_out/r2pdl; mkdir -p $out
L=paper_2007_01045_b200/libdapple.so
cp $L $out/new.so
timeout 900 python -m pytest tests/test_elementwise_gpu.py tests/test_executor_gpu.py tests/test_baseline_shapes_gpu.py tests/test_attention_gpu.py tests/test_lm_gpu.py tests/test_vgg_gpu.py tests/test_local_ranks_gpu.py -m gpu -q -x --timeout 300 --timeout-method thread -p no:cacheprovider -rf > $out/pytest.txt 2>&1
tail -1 $out/pytest.txt
for v in new old new old; do
  if [ $v = old ]; then cp ab/libdapple_old.so $L; else cp $out/new.so $L; fi
  timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e > $out/bert_$v.json 2> $out/bert_$v.err
  python -c "import json; d=json.load(open('$out/bert_$v.json')); print('bert $v', round(d['value'],2), d['clocks']['sm_mhz'], round(d['roofline']['frac'],4))"
  timeout 600 python bench.py --model gpt2-1.5b --steps 3 --warmup 3 --no-cpu --no-e2e > $out/gpt2_$v.json 2> $out/gpt2_$v.err
  python -c "import json; d=json.load(open('$out/gpt2_$v.json')); print('gpt2 $v', round(d['value'],2), d['clocks']['sm_mhz'], round(d['roofline']['frac'],4))"
done
for v in new old; do
  if [ $v = old ]; then cp ab/libdapple_old.so $L; else cp $out/new.so $L; fi
  timeout 600 python bench.py --model vgg19 --steps 5 --warmup 3 --no-cpu --no-e2e > $out/vgg_$v.json 2> $out/vgg_$v.err
  python -c "import json; d=json.load(open('$out/vgg_$v.json')); print('vgg $v', round(d['value'],2), d['clocks']['sm_mhz'])"
done
cp $out/new.so $L
