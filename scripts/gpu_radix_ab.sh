# A/B: screened top-k membership by radix select of the k-th key (LF_SEL_RADIX) vs O(n^2) ranks
show() { python -c "import json;d=json.load(open('$1'));print('$2', 'headline', round(d['value'],1), 'stateless', round(d['stateless']['value']), 'selplan_us', round(d['roofline_select']['select_plan_ms_per_call']*1e3,1))" 2>&1 | tail -1; }
for r in 1 0; do
  LF_NVCC_FLAGS=-DLF_SEL_RADIX=$r python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r$r.log 2>&1 || { tail -20 gpurun_out/build_r$r.log; exit 1; }
  if [ $r = 1 ]; then
    timeout 900 python -m pytest tests/test_gpu_select_plan.py tests/test_gpu_parity.py tests/test_gpu_paired.py -m gpu -q -x > gpurun_out/pytest_radix.log 2>&1; tail -2 gpurun_out/pytest_radix.log
  fi
  for c in c3 c5_s50 c5_s70; do
    timeout 300 python bench.py --config $c --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/rx${r}_$c.json 2> gpurun_out/rx${r}_$c.err
    show gpurun_out/rx${r}_$c.json "radix=$r $c"
  done
done
