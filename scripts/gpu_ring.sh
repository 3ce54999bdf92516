# K/V ring depth A/B (rebuilds the library per variant)
for fl in "" "-DLF_V7_KST=3 -DLF_V7_SLACK=0" "-DLF_V7_KST=3 -DLF_V7_VST=2" "-DLF_V7_KST=1 -DLF_V7_VST=4"; do
  LF_NVCC_FLAGS="$fl" python -c "from paper_2602_04789_b200.build import build; build(force=True)" > gpurun_out/b.log 2>&1 || { tail -5 gpurun_out/b.log; continue; }
  timeout 300 python -m pytest tests/test_gpu_kernels.py -m gpu -x -q -k "vs_oracle and 3" 2>&1 | tail -1
  for c in c2 c5_dense c3; do
    timeout 300 python bench.py --config $c --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/rg.json 2>/dev/null
    python -c "import json;d=json.load(open('gpurun_out/rg.json'));r=d['roofline'];print('[$fl] $c attn', round(r['achieved']), 'issued', round(r['issued_tflops']))" 2>&1 | tail -1
  done
done
