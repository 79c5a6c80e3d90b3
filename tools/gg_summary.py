"""One line per GEMM shape from a tools/gemm_graph_bench.py output file."""
import json
import sys

for line in open(sys.argv[1]):
    line = line.strip()
    if not line.startswith("{"):
        continue
    d = json.loads(line)
    if "gemm" in d:
        print(f"    {d['gemm']:12s} ours {d['ours_us']:7.2f} us  cublas {d['cublas_us']:7.2f} us")
    elif "sum_us" in d:
        print(f"    sum ours {d['sum_us']['ours']} cublas {d['sum_us']['cublas']}")
