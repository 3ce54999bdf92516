# plan tiles with (first block only, second block only) segment pairs inside each query tile
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py tests/test_gpu_paired.py tests/test_gpu_rollout.py tests/test_gpu_select_plan.py -m gpu -x -q 2>&1 | tail -3
for c in c3 c5_s50 c5_s70 c5_s85 c2; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/sub_$c.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/sub_$c.json'));r=d['roofline'];print('$c headline', round(d['value']), 'stateless', round(d['stateless']['value']), 'attn', round(r['achieved']), round(r['frac'],3), 'issued', round(r['issued_tflops']), 'attn us', round(r['attn_ms_per_call']*1e3,1))" 2>&1 | tail -1
done
