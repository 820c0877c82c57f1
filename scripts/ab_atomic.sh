python scripts/scatter_bench.py atomic
