python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
for c in c2 c5_dense; do for cfg in "7 0" "7 3" "7 4" "7 6" "7 8" "8 0" "8 4" "8 6" "8 8"; do
  set -- $cfg
  LF_TILE_VER=$1 LF_ATTN_POLY=$2 timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/vb.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/vb.json'));r=d['roofline'];print('ver $1 poly $2 $c attn', round(r['achieved']), 'issued', round(r['issued_tflops']), 'frac', round(r['frac'],3), 'err', d['device_errors'])" 2>&1 | tail -1
done; done
LF_ATTN_POLY=4 timeout 600 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x -k "TILE or 3" 2>&1 | tail -2
