# sweep environment settings over bench configs on one box:
#   SWEEP="LF_ATTN_POLY=0 LF_ATTN_POLY=4" CONFIGS="c2 c5_dense" bash scripts/gpu_sweep.sh
python -c "import __graft_entry__ as g; g.build()" > /dev/null
if [ -n "$TESTS" ]; then
  env $TESTENV timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$? >> gpurun_out/pytest_gpu.log
  tail -n 2 gpurun_out/pytest_gpu.log
fi
for sw in ${SWEEP:-NONE=0}; do
for c in ${CONFIGS:-c2}; do
  tag=$(echo $sw | tr '=,' '__')
  env ${sw//,/ } timeout 300 python bench.py --config $c --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/sw_${c}_$tag.json 2> gpurun_out/sw_${c}_$tag.err
  python -c "import json;d=json.load(open('gpurun_out/sw_${c}_$tag.json'));r=d['roofline'];s=d['roofline_select'];print('$sw $c', round(d['value'],1), 'TF/s', round(d['ms_per_chunk'],3), 'ms/chunk | attn', round(r['achieved'],1), round(r['frac'],3), round(r['attn_ms_per_call']*1e3,1),'us | pool', round(s['achieved']), 'GB/s', round(s['pool_ms_per_call']*1e3,1), 'us sel', round(s['select_plan_ms_per_call']*1e3,1), 'us err', d['device_errors'], '| issued', round(r.get('issued_tflops',0)))" || tail -n 5 gpurun_out/sw_${c}_$tag.err
done
done
