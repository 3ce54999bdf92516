python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py tests/test_gpu_paired.py tests/test_gpu_select_plan.py tests/test_gpu_rollout.py -m gpu -x -q 2>&1 | tail -1
PYTHONPATH=. timeout 300 python scripts/sel_micro.py plan
for c in c3 c5_s70 c2; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/pp.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/pp.json'));s=d['roofline_select'];print('$c headline', round(d['value']), 'stateless', round(d['stateless']['value']), 'selplan us', round(s['select_plan_ms_per_call']*1e3,1), 'stage', round(s['frac'],3))"
done
