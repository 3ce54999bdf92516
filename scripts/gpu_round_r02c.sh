# final evidence run of the round-2 tree (serial step order, PDL, graph-captured e2e): GPU tests
# + smoke, bench lines for every config, the reference arm, launch lists, ncu of attention and
# the selection, device timelines of the c2 / c5_s70 headline step
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 240 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$? >> gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q -rA > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$? >> gpurun_out/pytest_gpu.log
tail -n 3 gpurun_out/smoke.log gpurun_out/pytest_gpu.log
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref_c2.json 2> gpurun_out/bench_ref_c2.err
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
for c in c3 c4 c5_dense c5_s50 c5_s70 c5_s85; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
for c in c2 c3 c4 c5_dense c5_s50 c5_s70 c5_s85; do
  python -c "import json;d=json.load(open('gpurun_out/bench_$c.json'));r=d['roofline'];s=d['roofline_select'];e=d['e2e'];print('$c', d['query_tiles'], 'headline', round(d['value']), 'stateless', round(d['stateless']['value']), 'ms', round(d['ms_per_step'],3), 'attn', round(r['achieved']), round(r['frac'],3), 'issued', round(r['issued_tflops']), 'stage', round(s['frac'],3), 'pool', round(s['pool_frac'],3), 'selplan us', round(s['select_plan_ms_per_call']*1e3,1), 'e2e', round(e['value']), round(e['ms_per_chunk'],2), round(e['pcie_bound_ms_per_chunk'],2), d['clocks']['reasons'])" 2>&1 | tail -1
done
python -c "import json;d=json.load(open('gpurun_out/bench_ref_c2.json'));print('reference', d['value'], d['cpu_baseline']['kind'], d['cpu_baseline']['cores'])"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches_c5_s70.csv python bench.py --config c5_s70 --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_fwd -s 1 -c 1 -o gpurun_out/attn_c2 -f python bench.py --profile-launch --no-cpu-baseline --config c2 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:select_screen -s 2 -c 1 -o gpurun_out/select_c3 -f python bench.py --profile-launch --no-cpu-baseline --config c3 > /dev/null 2>&1
for c in c2 c5_s70; do
  LF_BENCH_TIMELINE=gpurun_out/timeline_$c.csv timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
done
ls -la gpurun_out/ | tail -40
