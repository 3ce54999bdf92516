python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py tests/test_gpu_paired.py -m gpu -x -q 2>&1 | tail -1
for rep in 1 2; do for c in c2 c4 c5_dense c3 c5_s50 c5_s70 c5_s85; do
  timeout 300 python bench.py --config $c --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/y.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/y.json'));r=d['roofline'];print('$rep $c headline', round(d['value']), 'attn', round(r['achieved']), 'issued', round(r['issued_tflops']))"
done; done
for p in 4 ; do LF_ATTN_POLY=$p timeout 300 python bench.py --config c2 --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/y.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/y.json'));r=d['roofline'];print('poly $p c2 attn', round(r['achieved']))"; done
