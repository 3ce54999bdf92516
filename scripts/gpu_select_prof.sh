# selection-stage breakdown at the sparse configs: per-kernel launch list and one
# ncu --set full capture each of select_cta_kernel / plan_tiles_cta_kernel at c5_s70
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
for c in c3 c5_s50 c5_s70; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches_$c.csv python bench.py --config $c --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:select_cta -s 2 -c 1 -o gpurun_out/select_c5_s70 -f python bench.py --profile-launch --no-cpu-baseline --config c5_s70 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:plan_tiles -s 2 -c 1 -o gpurun_out/plan_c5_s70 -f python bench.py --profile-launch --no-cpu-baseline --config c5_s70 > /dev/null 2>&1
ls -la gpurun_out/
