# A/B: attention with one vs two Q buffers (LF_V7_QST), bench lines per config; parity tests on QST=2
show() { python -c "import json;d=json.load(open('$1'));r=d['roofline'];print('$2', 'headline', round(d['value'],1), 'attn', round(r['achieved']), round(r['frac'],3), 'issued', round(r['issued_tflops']))" 2>&1 | tail -1; }
for q in 1 2; do
  LF_NVCC_FLAGS=-DLF_V7_QST=$q python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_q$q.log 2>&1 || { tail -30 gpurun_out/build_q$q.log; exit 1; }
  for c in c2 c3 c5_s50 c5_s70 c5_dense; do
    LF_NVCC_FLAGS=-DLF_V7_QST=$q timeout 300 python bench.py --config $c --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/q${q}_$c.json 2> gpurun_out/q${q}_$c.err
    show gpurun_out/q${q}_$c.json "q$q $c"
  done
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kernels.py tests/test_gpu_paired.py tests/test_gpu_qtiles.py -m gpu -x -q > gpurun_out/pytest_q2.log 2>&1; tail -2 gpurun_out/pytest_q2.log
# e2e stability: per-iteration times, host enqueue time and allocator events of the e2e legs
for c in c2 c3 c2 c3; do
  LF_BENCH_TRACE=1 timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/tr_$c.json 2>> gpurun_out/tr_$c.err
  python -c "import json;d=json.load(open('gpurun_out/tr_$c.json'));print('$c e2e', round(d['e2e']['value']), round(d['e2e']['ms_per_chunk'],2))"
done
nproc; uptime; cat /proc/loadavg
