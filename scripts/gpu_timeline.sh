python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
for c in c2 c5_s70; do
  LF_BENCH_TIMELINE=gpurun_out/timeline_$c.csv timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/tl_$c.json 2> gpurun_out/tl_$c.err
  python -c "import json;d=json.load(open('gpurun_out/tl_$c.json'));print('$c headline', round(d['value']), 'ms/chunk', round(d['ms_per_step'],3), 'stateless', round(d['stateless']['value']))"
done
