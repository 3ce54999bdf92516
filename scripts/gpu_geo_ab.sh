python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
for rep in 1 2; do for c in c5_s70 c3; do for q in blocks paired; do
  LF_QTILE=$q timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/geo_${c}_$q.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/geo_${c}_$q.json'));r=d['roofline'];s=d['roofline_select'];print('$c $q headline', round(d['value']), 'stateless', round(d['stateless']['value']), 'attn us', round(r['attn_ms_per_call']*1e3,1), 'selplan us', round(s['select_plan_ms_per_call']*1e3,1))" 2>&1 | tail -1
done; done; done
