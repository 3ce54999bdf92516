# A/B of the Q double buffer (LF_NVCC_FLAGS rebuilds the library with the single-buffer variant)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_paired.py -m gpu -x -q 2>&1 | tail -2
for c in c2 c4 c5_dense c3 c5_s50; do
  timeout 300 python bench.py --config $c --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/qst2_$c.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/qst2_$c.json'));r=d['roofline'];print('QST2 $c headline', round(d['value']), 'attn', round(r['achieved']), 'issued', round(r['issued_tflops']))"
done
LF_NVCC_FLAGS="-DLF_V7_QST=1" python -c "from paper_2602_04789_b200.build import build; build(force=True)" > gpurun_out/build1.log 2>&1 || tail gpurun_out/build1.log
for c in c2 c4 c5_dense c3 c5_s50; do
  LF_NVCC_FLAGS="-DLF_V7_QST=1" timeout 300 python bench.py --config $c --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/qst1_$c.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/qst1_$c.json'));r=d['roofline'];print('QST1 $c headline', round(d['value']), 'attn', round(r['achieved']), 'issued', round(r['issued_tflops']))"
done
