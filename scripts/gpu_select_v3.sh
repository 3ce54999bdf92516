# screened selection: GPU selection/parity tests, then select+plan time per config with the
# screen (default) and with every score exact (LF_SELECT_EXACT=1), and one launch list at c5_s70
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_select_plan.py tests/test_gpu_parity.py tests/test_gpu_rollout.py tests/test_gpu_paired.py -m gpu -x -q > gpurun_out/pytest_sel.log 2>&1; tail -3 gpurun_out/pytest_sel.log
for c in c2 c3 c5_s50 c5_s70; do for ex in 0 1; do
  if [ $ex = 1 ]; then export LF_SELECT_EXACT=1; else unset LF_SELECT_EXACT; fi
  timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/sx_${c}_$ex.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/sx_${c}_$ex.json'));s=d['roofline_select'];print('$c exact=$ex headline', round(d['value']), 'stateless', round(d['stateless']['value']), 'selplan us', round(s['select_plan_ms_per_call']*1e3,1), 'stage', round(s['frac'],3))" 2>&1 | tail -1
done; done
unset LF_SELECT_EXACT
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches_sel_c5_s70.csv python bench.py --config c5_s70 --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
grep -i "select\|plan_tiles\|pair_q\|pool_frames" gpurun_out/launches_sel_c5_s70.csv | awk -F'","' '{print $5, $(NF)}' | head
