python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for c in c3 c5_s70 c5_s85; do for m in blocks paired; do
  LF_QTILE=$m timeout 300 python bench.py --config $c --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/q.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/q.json'));r=d['roofline'];print('$m $c headline', round(d['value']), 'attn', round(r['achieved']), 'us', round(r['attn_ms_per_call']*1e3,1), 'selplan', round(d['roofline_select']['select_plan_ms_per_call']*1e3,1))"
done; done
