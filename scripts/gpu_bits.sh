python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_paired.py tests/test_gpu_select_plan.py tests/test_gpu_rollout.py tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -2
for c in c5_s50 c5_s70; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bb.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/bb.json'));s=d['roofline_select'];print('$c headline', round(d['value']), 'stateless', round(d['stateless']['value']), 'selplan us', round(s['select_plan_ms_per_call']*1e3,1), 'stage', round(s['frac'],3))"
done
