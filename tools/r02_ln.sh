#!/bin/bash
out=gpurun_out/r2ln; mkdir -p $out
timeout 600 python -m pytest tests/test_elementwise_gpu.py tests/test_executor_gpu.py -m gpu -q -x --timeout 300 --timeout-method thread -p no:cacheprovider -rf > $out/pytest.txt 2>&1
tail -1 $out/pytest.txt
timeout 100 python tools/attn_bench.py 2>&1 | tail -5
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu > $out/bert.json 2> $out/bert.err
python -c "import json; d=json.load(open('$out/bert.json')); print('bert', round(d['value'],2), d['clocks']['sm_mhz'], [(k['kernel'], round(k['seconds']*1e3,2)) for k in d['kernels'] if 'layernorm' in k['kernel']])"
cmd="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-profile"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:'layernorm|ln_' -c 60 --csv --log-file $out/ln.csv $cmd > $out/ncu.log 2>&1; echo "ncu rc=$?"
python tools/launch_shares.py $out/ln.csv
