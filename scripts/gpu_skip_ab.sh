# A/B: masked-half skip (working tree) vs the round-2 final kernel (scripts/v7_base.cuh)
cp paper_2602_04789_b200/csrc/attn_sm100_v7.cuh /tmp/v7_skip.cuh
for rep in 1 2; do for var in skip base; do
  if [ $var = base ]; then cp scripts/v7_base.cuh paper_2602_04789_b200/csrc/attn_sm100_v7.cuh; else cp /tmp/v7_skip.cuh paper_2602_04789_b200/csrc/attn_sm100_v7.cuh; fi
  python -c "from paper_2602_04789_b200.build import build; build(force=True)" > /dev/null 2>&1
  for c in c2 c5_dense c3 c5_s50 c5_s70; do
    timeout 300 python bench.py --config $c --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/ab.json 2>/dev/null
    python -c "import json;d=json.load(open('gpurun_out/ab.json'));r=d['roofline'];print('$rep $var $c headline', round(d['value']), 'attn', round(r['achieved']))"
  done
done; done
cp /tmp/v7_skip.cuh paper_2602_04789_b200/csrc/attn_sm100_v7.cuh
