python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
LF_TILE_VER=9 timeout 120 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
LF_TILE_VER=9 timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py tests/test_gpu_qtiles.py -m gpu -x -q 2>&1 | tail -4
for c in c2 c5_dense c3 c5_s50; do for v in 7 9; do
  LF_TILE_VER=$v timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/v${v}_$c.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/v${v}_$c.json'));r=d['roofline'];print('v$v $c headline', round(d['value']), 'attn', round(r['achieved']), 'issued', round(r['issued_tflops']), 'frac', round(r['frac'],3), 'err', d['device_errors'])" 2>&1 | tail -1
done; done
