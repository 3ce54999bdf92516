# compare attention kernel versions on the same box
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$? >> gpurun_out/pytest_gpu.log
tail -n 2 gpurun_out/pytest_gpu.log
for ver in ${VERS:-3 2}; do
for c in ${CONFIGS:-c2 c2h16 c5_dense c5_s50 c3}; do
  LF_ATTN_VER=$ver timeout 300 python bench.py --config $c --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${c}_v$ver.json 2> gpurun_out/bench_${c}_v$ver.err
  python -c "import json;d=json.load(open('gpurun_out/bench_${c}_v$ver.json'));r=d['roofline'];s=d['roofline_select'];print('v$ver $c', round(d['value'],1), 'TF/s step', round(d['ms_per_chunk'],3), 'ms/chunk | attn', round(r['achieved'],1), round(r['frac'],3), round(r['attn_ms_per_call']*1e3,1),'us | pool', round(s['achieved']), 'GB/s', round(s['pool_ms_per_call']*1e3,1), 'us sel', round(s['select_plan_ms_per_call']*1e3,1), 'us')" || tail -n 5 gpurun_out/bench_${c}_v$ver.err
done
done
if [ -n "$NCU" ]; then
LF_ATTN_VER=${NCU_VER:-3} timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_fwd -s 1 -c 1 -o gpurun_out/attn_cmp python bench.py --profile-launch --no-cpu-baseline --config ${NCU_CONFIG:-c2} > gpurun_out/ncu_attn.log 2>&1
fi
