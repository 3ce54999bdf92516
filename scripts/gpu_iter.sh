# quick iteration: parity tests + a few bench configs + one ncu capture of the attention kernel
set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$? >> gpurun_out/pytest_gpu.log
tail -n 3 gpurun_out/pytest_gpu.log
for c in ${CONFIGS:-c2 c5_s50 c5_dense}; do
  timeout 300 python bench.py --config $c --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  python -c "import json;d=json.load(open('gpurun_out/bench_$c.json'));r=d['roofline'];s=d['roofline_select'];print('$c', round(d['value'],1), 'TF/s step', round(d['ms_per_chunk'],3), 'ms/chunk | attn', round(r['achieved'],1), round(r['frac'],3), round(r['attn_ms_per_call']*1e3,1),'us | pool', round(s['achieved']), 'GB/s', round(s['pool_ms_per_call']*1e3,1), 'us sel', round(s['select_plan_ms_per_call']*1e3,1), 'us')" || tail -n 20 gpurun_out/bench_$c.err
done
if [ -n "$NCU" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_fwd -s 1 -c 1 -o gpurun_out/attn_iter python bench.py --profile-launch --no-cpu-baseline --config ${NCU_CONFIG:-c2} > gpurun_out/ncu_attn.log 2>&1
fi
if [ -n "$CMP_V1" ]; then
  LF_ATTN_V1=1 timeout 300 python bench.py --config c2 --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2_v1.json 2>&1
  python -c "import json;d=json.load(open('gpurun_out/bench_c2_v1.json'));r=d['roofline'];print('v1 c2', round(d['value'],1), round(r['achieved'],1), round(r['frac'],3))"
fi
