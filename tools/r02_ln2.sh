#!/bin/bash
# LayerNorm packed-math A/B: new lib vs ab/libdapple_old.so (same box)
out=gpurun_out/r2ln2; mkdir -p $out
L=paper_2007_01045_b200/libdapple.so
cp $L $out/new.so
timeout 600 python -m pytest tests/test_elementwise_gpu.py tests/test_executor_gpu.py tests/test_baseline_shapes_gpu.py -m gpu -q -x --timeout 300 --timeout-method thread -p no:cacheprovider -rf > $out/pytest.txt 2>&1
tail -1 $out/pytest.txt
for v in new old new old; do
  if [ $v = old ]; then cp ab/libdapple_old.so $L; else cp $out/new.so $L; fi
  echo "== $v"; timeout 120 python tools/elementwise_graph_bench.py 2>&1 | tail -5
  timeout 120 python tools/elementwise_graph_bench.py --h 1600 --rows 1024 2>&1 | head -2
done
for v in new old new old; do
  if [ $v = old ]; then cp ab/libdapple_old.so $L; else cp $out/new.so $L; fi
  timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e > $out/bert_$v.json 2> $out/bert_$v.err
  python -c "import json; d=json.load(open('$out/bert_$v.json')); print('bert $v', round(d['value'],2), d['clocks']['sm_mhz'], [(k['kernel'], round(k['seconds']*1e3,2)) for k in d['kernels'] if 'layernorm' in k['kernel']])"
done
cp $out/new.so $L
cmd="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-profile"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:'layernorm|ln_' -c 40 --csv --log-file $out/ln.csv $cmd > $out/ncu.log 2>&1; echo "ncu rc=$?"
python tools/launch_shares.py $out/ln.csv
