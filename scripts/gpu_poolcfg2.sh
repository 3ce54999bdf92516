python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
for c in c2 c4; do for cfg in 2x4 4x4 4x8 8x8; do
  LF_POOL_CFG=$cfg timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/pc.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/pc.json'));s=d['roofline_select'];print('$c $cfg pool us', round(s['pool_ms_per_call']*1e3,2), 'pool frac', round(s['pool_frac'],3), 'stateless', round(d['stateless']['value']))"
done; done
