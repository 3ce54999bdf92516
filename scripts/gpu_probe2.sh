python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for c in c2 c5_dense; do for dbg in 0 1 4 5 6 7; do
  LF_ATTN_DEBUG=$dbg timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/pr.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/pr.json'));r=d['roofline'];print('$c dbg $dbg attn issued', round(r['issued_tflops']), 'us', round(r['attn_ms_per_call']*1e3,1))"
done; done
