#!/bin/bash
# early triggers in the conv / LM / SGD kernels too: new lib vs ab/libdapple_old.so
out=gpurun_out/r2pdl2; mkdir -p $out
L=paper_2007_01045_b200/libdapple.so
cp $L $out/new.so
timeout 900 python -m pytest tests/test_conv_gpu.py tests/test_vgg_gpu.py tests/test_lm_gpu.py tests/test_executor_gpu.py tests/test_elementwise_gpu.py -m gpu -q -x --timeout 300 --timeout-method thread -p no:cacheprovider -rf > $out/pytest.txt 2>&1
tail -1 $out/pytest.txt
for v in new old new old; do
  if [ $v = old ]; then cp ab/libdapple_old.so $L; else cp $out/new.so $L; fi
  for m in vgg19 amoebanet36 gpt2-1.5b; do
    timeout 600 python bench.py --model $m --steps 5 --warmup 3 --no-cpu --no-e2e > $out/${m}_$v.json 2> $out/${m}_$v.err
    python -c "import json; d=json.load(open('$out/${m}_$v.json')); print('$m $v', round(d['value'],2), d['clocks']['sm_mhz'])"
  done
done
cp $out/new.so $L
