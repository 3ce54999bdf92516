for nst in 3 6 8; do
  touch paper_2602_04789_b200/csrc/lfattn.cu
  LF_NVCC_FLAGS="-DLF_POOL_NST=$nst" python -c "import __graft_entry__ as g; g.build()" > /dev/null
  timeout 300 python bench.py --config c2 --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/pool_nst$nst.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/pool_nst$nst.json'));s=d['roofline_select'];print('NST $nst', round(s['achieved']), round(s['pool_ms_per_call']*1e3,1))"
done
