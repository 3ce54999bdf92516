python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_paired.py tests/test_gpu_qtiles.py tests/test_gpu_kernels.py -m gpu -x -q -s 2>&1 | grep -E "passed|failed|Error|issued|assert" | tail -8
for c in c3 c5_s50 c5_s70 c5_s85 c2; do for m in blocks paired; do
  LF_QTILE=$m timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/q_${m}_$c.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/q_${m}_$c.json'));r=d['roofline'];print('$m $c headline', round(d['value']), 'attn', round(r['achieved']), 'issued', round(r['issued_tflops']), 'frac', round(r['frac'],3), 'us', round(r['attn_ms_per_call']*1e3,1), 'selplan', round(d['roofline_select']['select_plan_ms_per_call']*1e3,1), 'err', d['device_errors'], d['query_tiles'])" 2>&1 | tail -1
done; done
