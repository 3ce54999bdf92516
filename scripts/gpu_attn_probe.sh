# attention ceiling probes (LF_ATTN_DEBUG: 0 normal, 1 no softmax math, 3 no softmax + no K/V reloads)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
for c in ${1:-c2 c5_dense c3}; do for dbg in 0 1 3; do
  LF_ATTN_DEBUG=$dbg timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/probe_${c}_$dbg.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/probe_${c}_$dbg.json'));r=d['roofline'];print('$c dbg $dbg attn', round(r['achieved']), 'issued', round(r['issued_tflops']), 'us', round(r['attn_ms_per_call']*1e3,1))"
done; done
