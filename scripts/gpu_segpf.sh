python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kernels.py -m gpu -x -q 2>&1 | tail -1
for c in c3 c5_s70 c5_s50 c2 c5_dense; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/pf.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/pf.json'));r=d['roofline'];print('$c headline', round(d['value']), 'attn', round(r['achieved']), 'issued', round(r['issued_tflops']), 'attn us', round(r['attn_ms_per_call']*1e3,1))" 2>&1 | tail -1
done
