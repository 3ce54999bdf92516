# quick GPU iteration: build, the named pytest files (default: the whole GPU suite), bench lines
# usage: bash scripts/gpu_quick.sh "<pytest targets>" "<bench configs>"
T=${1:-tests}
C=${2:-c2 c3}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 1200 python -m pytest $T -m gpu -x -q -rA -s > gpurun_out/pytest_quick.log 2>&1; echo pytest rc=$? >> gpurun_out/pytest_quick.log
grep -E "passed|failed|error|margin|rc=" gpurun_out/pytest_quick.log | tail -15
for c in $C; do
  timeout 300 python bench.py --config $c --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  python -c "import json;d=json.load(open('gpurun_out/bench_$c.json'));r=d['roofline'];s=d['roofline_select'];print('$c', d['config']['query_tiles'], 'headline', round(d['value']), 'attn', round(r['achieved']), round(r['frac'],3), 'pool', round(s['frac'],3), 'pool_us', round(s['pool_ms_per_call']*1e3,1), 'selplan_us', round(s['select_plan_ms_per_call']*1e3,1), 'e2e', round(d['e2e']['value']))" 2>&1 | tail -1
done
