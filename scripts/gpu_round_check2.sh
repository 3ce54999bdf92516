# full GPU suite + smoke + bench lines for every config with the automatic query-tile geometry
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 240 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$? >> gpurun_out/smoke.log
timeout 900 python -m pytest tests -m gpu -x -q -rA > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$? >> gpurun_out/pytest_gpu.log
tail -n 3 gpurun_out/smoke.log gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 50 --warmup 5 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
for c in c3 c4 c5_dense c5_s50 c5_s70 c5_s85; do
  timeout 300 python bench.py --config $c --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
for c in c2 c3 c4 c5_dense c5_s50 c5_s70 c5_s85; do
  python -c "import json;d=json.load(open('gpurun_out/bench_$c.json'));r=d['roofline'];s=d['roofline_select'];print('$c', d['config']['query_tiles'], 'headline', round(d['value']), 'attn', round(r['achieved']), round(r['frac'],3), 'pool', round(s['frac'],3), 'e2e', round(d['e2e']['value']))" 2>&1 | tail -1
done
