# Round profiles: bench line, ncu launch list of the bench command, ncu --set full
# of the step kernel and of both scatter pipelines (outputs in gpurun_out/).
set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_r1f.csv python bench.py --steps 10 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/bench_under_ncu.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:step_kernel -s 3 -c 1 -o gpurun_out/step_full_r1f python scripts/prof_step.py --batch 4096 > gpurun_out/ncu_step.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"sc_atomic_hot" -c 2 -o gpurun_out/scatter_atomic_r1f python scripts/scatter_bench.py atomic > gpurun_out/ncu_sc.log 2>&1
ls -la gpurun_out
