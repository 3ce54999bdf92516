# re-entry check of the current tree: build, smoke, full GPU suite, bench lines of the sparse configs
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 240 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$? >> gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q -rA > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$? >> gpurun_out/pytest_gpu.log
tail -n 3 gpurun_out/smoke.log gpurun_out/pytest_gpu.log
grep -E "^(FAILED|ERROR)" gpurun_out/pytest_gpu.log | head
for c in c2 c3 c5_s50 c5_s70 c5_s85; do
  timeout 300 python bench.py --config $c --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  python -c "import json;d=json.load(open('gpurun_out/bench_$c.json'));r=d['roofline'];s=d['roofline_select'];print('$c', d['config']['query_tiles'], 'headline', round(d['value']), 'attn', round(r['achieved']), round(r['frac'],3), 'issued', round(r['issued_tflops']), 'stage', round(s['frac'],3), 'selplan_us', round(s['select_plan_ms_per_call']*1e3,1), 'e2e', round(d['e2e']['value']))" 2>&1 | tail -1
done
