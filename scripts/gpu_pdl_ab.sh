# PDL on/off A/B (serial step order, graph-captured e2e), then the full GPU suite on the PDL build
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
show() { python -c "import json;d=json.load(open('$1'));r=d['roofline'];s=d['roofline_select'];print('$2', 'headline', round(d['value'],1), 'ms', round(d['ms_per_step'],4), 'stateless', round(d['stateless']['value']), 'attn', round(r['achieved']), 'selplan_us', round(s['select_plan_ms_per_call']*1e3,1), 'e2e', round(d['e2e']['value']), round(d['e2e']['ms_per_chunk'],3), 'bound', round(d['e2e']['pcie_bound_ms_per_chunk'],3))" 2>&1 | tail -1; }
for c in c2 c3 c5_s70; do
  for pdl in 1 0; do
    LF_PDL=$pdl LF_BENCH_TRACE=1 timeout 300 python bench.py --config $c --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/pdl${pdl}_$c.json 2> gpurun_out/pdl${pdl}_$c.err
    show gpurun_out/pdl${pdl}_$c.json "pdl$pdl $c"
  done
done
LF_BENCH_TIMELINE=gpurun_out/timeline_c2_pdl.csv timeout 300 python bench.py --config c2 --steps 5 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 240 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$? >> gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$? >> gpurun_out/pytest_gpu.log
tail -n 2 gpurun_out/smoke.log gpurun_out/pytest_gpu.log
