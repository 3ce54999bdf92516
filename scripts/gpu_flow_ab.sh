# A/B of the rollout step order (LF_BENCH_FLOW): overlap / serial / prio / prio2, headline lines
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
for c in c2 c3 c5_s70; do
  for fl in overlap serial prio prio2; do
    LF_BENCH_FLOW=$fl timeout 300 python bench.py --config $c --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/flow_${c}_$fl.json 2> gpurun_out/flow_${c}_$fl.err
    python -c "import json;d=json.load(open('gpurun_out/flow_${c}_$fl.json'));print('$c $fl headline', round(d['value'],1), 'ms', round(d['ms_per_step'],4), 'e2e', round(d['e2e']['value']))" 2>&1 | tail -1
  done
done
for fl in overlap prio2; do
  LF_BENCH_FLOW=$fl LF_BENCH_TIMELINE=gpurun_out/timeline_c2_$fl.csv timeout 300 python bench.py --config c2 --steps 5 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
done
