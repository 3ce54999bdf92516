# A/B: MMA-warp per-set state in scalars (new) vs x-indexed arrays in local memory (old, gpurun_out/ab_old_v7.cuh)
show() { python -c "import json;d=json.load(open('$1'));r=d['roofline'];print('$2', 'headline', round(d['value'],1), 'attn', round(r['achieved']), round(r['frac'],3))" 2>&1 | tail -1; }
run() {
  python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$1.log 2>&1 || { tail -20 gpurun_out/build_$1.log; exit 1; }
  for c in c2 c5_dense c3 c2; do
    timeout 300 python bench.py --config $c --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/mr_$1_$c.json 2>/dev/null
    show gpurun_out/mr_$1_$c.json "$1 $c"
  done
}
run new
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kernels.py tests/test_gpu_paired.py tests/test_gpu_qtiles.py -m gpu -x -q > gpurun_out/pytest_mr.log 2>&1; tail -1 gpurun_out/pytest_mr.log
cp scripts/ab_old_v7.cuh paper_2602_04789_b200/csrc/attn_sm100_v7.cuh
run old
