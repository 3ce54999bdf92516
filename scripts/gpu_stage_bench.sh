# full GPU tests, then the bench lines (stage numbers) of the sparse configs and c2
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
for c in c2 c3 c5_s50 c5_s70 c5_s85; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  python -c "import json;d=json.load(open('gpurun_out/bench_$c.json'));r=d['roofline'];s=d['roofline_select'];print('$c', d['query_tiles'], 'headline', round(d['value']), 'stateless', round(d['stateless']['value']), 'attn', round(r['achieved']), round(r['frac'],3), 'stage', round(s['frac'],3), 'selplan us', round(s['select_plan_ms_per_call']*1e3,1), 'e2e', round(d['e2e']['value']))" 2>&1 | tail -1
done
