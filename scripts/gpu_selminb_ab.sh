# A/B: selection kernel register budget (LF_SEL_MINB resident CTAs per SM)
for b in 7 4 10; do
  LF_NVCC_FLAGS=-DLF_SEL_MINB=$b python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_b$b.log 2>&1 || exit 1
  for c in c3 c5_s70; do
    timeout 300 python bench.py --config $c --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/mb${b}_$c.json 2>/dev/null
    python -c "import json;d=json.load(open('gpurun_out/mb${b}_$c.json'));print('minb=$b $c', round(d['value'],1), 'selplan_us', round(d['roofline_select']['select_plan_ms_per_call']*1e3,1))"
  done
done
