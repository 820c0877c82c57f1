# Round-2 evidence (outputs in gpurun_out/), in parts so each call's output stays small:
#   bash scripts/prof_round2.sh bench | step | scatter
set -x
case "$1" in
bench)
  python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
  python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
  python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_r2.csv python bench.py --steps 10 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/bench_under_ncu.log 2>&1
  # compute-sanitizer runs (profiles/sanitizer_r2) are no longer possible: the
  # pool closed the tool after it left GPUs needing a reset
  ;;
step)
  ncu --set full --import-source on --clock-control none -k regex:step_kernel -s 3 -c 1 -o gpurun_out/step_b4096_r2 python scripts/prof_step.py --batch 4096 > gpurun_out/ncu_step.log 2>&1
  ncu --set full --import-source on --clock-control none -k regex:step_kernel -s 3 -c 1 -o gpurun_out/step_b1024_r2 python scripts/prof_step.py --batch 1024 >> gpurun_out/ncu_step.log 2>&1
  ncu --set full --import-source on --clock-control none -k regex:step_kernel -s 3 -c 1 -o gpurun_out/step_large512_r2 python scripts/prof_step.py --large --batch 512 >> gpurun_out/ncu_step.log 2>&1
  ;;
scatter)
  ncu --set full --import-source on --clock-control none -k regex:sc_det_owner -s 1 -c 1 -o gpurun_out/det_owner_zipf_r2 python scripts/prof_scatter.py det zipf 2 > gpurun_out/ncu_sc.log 2>&1
  ncu --set full --import-source on --clock-control none -k regex:sc_det_owner -s 1 -c 1 -o gpurun_out/det_owner_uniform_r2 python scripts/prof_scatter.py det uniform 2 >> gpurun_out/ncu_sc.log 2>&1
  ncu --set full --import-source on --clock-control none -k regex:sc_atomic_hot -s 1 -c 1 -o gpurun_out/atomic_zipf_r2 python scripts/prof_scatter.py atomic zipf 2 >> gpurun_out/ncu_sc.log 2>&1
  ;;
esac
ls -la gpurun_out
