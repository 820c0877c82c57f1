for c in 0; do python scripts/scatter_bench.py atomic; done
