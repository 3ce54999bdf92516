# dynamic vs static item schedule of the tile attention kernel (run via gpurun)
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 300 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_qtiles.py -x -q 2>&1 | tail -3
for c in c3 c5_s70 c2 c5_dense; do
  for m in dyn static; do
    if [ $m = static ]; then export LF_ATTN_STATIC=1; else unset LF_ATTN_STATIC; fi
    timeout 300 python bench.py --config $c --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/sch_${m}_$c.json 2>gpurun_out/sch_${m}_$c.err
    python -c "import json;d=json.load(open('gpurun_out/sch_${m}_$c.json'));r=d['roofline'];print('$c $m headline', round(d['value']), 'attn', round(r['achieved']), round(r['frac'],3), 'us', round(r['attn_ms_per_call']*1e3,1))" 2>&1 | tail -1
  done
done
unset LF_ATTN_STATIC
