# A/B of the pooling kernel's (consumer groups x ring stages) at c2 and c5_dense (run via gpurun)
python -c "import __graft_entry__ as g; g.build()" > /dev/null
for cfg in 2x4 4x4 2x4 4x4; do
  for c in c2 c3; do
    LF_POOL_CFG=$cfg timeout 300 python bench.py --config $c --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/pool_${cfg}_$c.json 2>gpurun_out/pool_${cfg}_$c.err
    python -c "import json;d=json.load(open('gpurun_out/pool_${cfg}_$c.json'));s=d['roofline_select'];print('$cfg $c', round(s['achieved']), round(s['frac'],3), round(s['pool_ms_per_call']*1e3,1), 'headline', round(d['value']))"
  done
done
