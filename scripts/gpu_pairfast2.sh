# pairing: overlaps over the SMs, warp-per-block rounds, proposals kept while their partner is free
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_paired.py tests/test_gpu_select_plan.py tests/test_gpu_rollout.py tests/test_gpu_qtiles.py -m gpu -q -x > gpurun_out/pytest_pf2.log 2>&1; echo pytest rc=$? >> gpurun_out/pytest_pf2.log
tail -3 gpurun_out/pytest_pf2.log; grep -E "FAILED|Error" gpurun_out/pytest_pf2.log | head -5
show() { python -c "import json;d=json.load(open('$1'));r=d['roofline'];print('$2', d['query_tiles'][:12], 'headline', round(d['value'],1), 'ms', round(d['ms_per_step'],4), 'attn', round(r['achieved']), 'selplan_us', round(d['roofline_select']['select_plan_ms_per_call']*1e3,1))" 2>&1 | tail -1; }
for c in c5_s50 c5_s70; do
  timeout 300 python bench.py --config $c --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/pf2_$c.json 2> gpurun_out/pf2_$c.err
  show gpurun_out/pf2_$c.json "pairfast2 $c"
done
LF_QTILE=paired timeout 300 python bench.py --config c3 --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/pf2p_c3.json 2> gpurun_out/pf2p_c3.err
show gpurun_out/pf2p_c3.json "pairfast2 forced-paired c3"
LF_BENCH_TIMELINE=gpurun_out/timeline_c5_s70_pf2.csv timeout 300 python bench.py --config c5_s70 --steps 5 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
