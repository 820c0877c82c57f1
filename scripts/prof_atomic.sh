ncu --set full --import-source on --clock-control none -k regex:"sc_atomic_hot" -c 2 -o gpurun_out/scatter_atomic_r1c python scripts/scatter_bench.py atomic > gpurun_out/ncu_sc.log 2>&1
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
