# A/B: attention epilogue releasing O before the global stores (LF_V7_EARLY_O), parity on the new build
show() { python -c "import json;d=json.load(open('$1'));r=d['roofline'];print('$2', 'headline', round(d['value'],1), 'attn', round(r['achieved']), round(r['frac'],3), 'issued', round(r['issued_tflops']))" 2>&1 | tail -1; }
for e in 0 1; do
  LF_NVCC_FLAGS=-DLF_V7_EARLY_O=$e python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_e$e.log 2>&1 || { tail -20 gpurun_out/build_e$e.log; exit 1; }
  for c in c2 c3 c5_s50 c5_dense; do
    timeout 300 python bench.py --config $c --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/eo${e}_$c.json 2> gpurun_out/eo${e}_$c.err
    show gpurun_out/eo${e}_$c.json "earlyO=$e $c"
  done
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kernels.py tests/test_gpu_paired.py tests/test_gpu_qtiles.py tests/test_gpu_rollout.py -m gpu -x -q > gpurun_out/pytest_eo.log 2>&1; tail -2 gpurun_out/pytest_eo.log
