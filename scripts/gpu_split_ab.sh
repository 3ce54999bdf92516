python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
for c in c3 c5_s70 c5_s50 c2; do for sp in 0 2 3; do
  LF_ATTN_SPLIT=$sp timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/sp.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/sp.json'));r=d['roofline'];print('$c split=$sp headline', round(d['value']), 'attn', round(r['achieved']), 'issued', round(r['issued_tflops']), 'attn us', round(r['attn_ms_per_call']*1e3,1))" 2>&1 | tail -1
done; done
