# selection without the frame list (rollout default): parity tests and bench lines
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_select_plan.py tests/test_gpu_rollout.py tests/test_gpu_paired.py tests/test_gpu_kernels.py -m gpu -q -x > gpurun_out/pytest_nf.log 2>&1; echo pytest rc=$? >> gpurun_out/pytest_nf.log
tail -3 gpurun_out/pytest_nf.log
show() { python -c "import json;d=json.load(open('$1'));r=d['roofline'];print('$2', 'headline', round(d['value'],1), 'ms', round(d['ms_per_step'],4), 'attn', round(r['achieved']), 'e2e', round(d['e2e']['value']), round(d['e2e']['ms_per_chunk'],3))" 2>&1 | tail -1; }
for c in c2 c2 c3 c5_s70; do
  timeout 300 python bench.py --config $c --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/nf_$c.json 2> gpurun_out/nf_$c.err
  show gpurun_out/nf_$c.json "noframes $c"
done
LF_BENCH_TIMELINE=gpurun_out/timeline_c2_nf.csv timeout 300 python bench.py --config c2 --steps 5 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
