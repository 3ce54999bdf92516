# block-aligned vs 128-row query tiles (run via gpurun): GPU tests, then A/B per config
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 600 python -m pytest tests/test_gpu_qtiles.py -x -q 2>&1 | tail -15
for c in c3 c5_s50 c5_s70 c5_s85 c2; do
  for m in rows blocks; do
    LF_QTILE=$m timeout 300 python bench.py --config $c --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/qt_${m}_$c.json 2>gpurun_out/qt_${m}_$c.err
    python -c "import json;d=json.load(open('gpurun_out/qt_${m}_$c.json'));r=d['roofline'];print('$c $m headline', round(d['value']), 'attn', round(r['achieved']), round(r['frac'],3), 'us', round(r['attn_ms_per_call']*1e3,1), 'issued', round(r['issued_tflops']))" 2>&1 | tail -1
  done
done
