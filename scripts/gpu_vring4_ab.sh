# A/B: V ring 4 stages (fits with the 512-byte alignment slack) vs 3
show() { python -c "import json;d=json.load(open('$1'));r=d['roofline'];print('$2', 'headline', round(d['value'],1), 'attn', round(r['achieved']), round(r['frac'],3))" 2>&1 | tail -1; }
for v in 4 3; do
  LF_NVCC_FLAGS=-DLF_V7_VST=$v python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_v$v.log 2>&1 || { tail -20 gpurun_out/build_v$v.log; exit 1; }
  for c in c2 c5_dense c3 c2; do
    timeout 300 python bench.py --config $c --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/vr${v}_$c.json 2>/dev/null
    show gpurun_out/vr${v}_$c.json "V$v $c"
  done
  if [ $v = 4 ]; then timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/pytest_v4.log 2>&1; tail -1 gpurun_out/pytest_v4.log; fi
done
