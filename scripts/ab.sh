# A/B the prebuilt libraries ab/<name>.so on one box (run via gpurun):
#   LIBS="old new" CONFIGS="c2 c5_dense" ROUNDS=2 bash scripts/ab.sh
for r in $(seq ${ROUNDS:-2}); do
for v in ${LIBS:-old new}; do
  cp ab/$v.so paper_2602_04789_b200/_lib/liblfattn.so
  for c in ${CONFIGS:-c2}; do
    env $ABENV timeout 300 python bench.py --config $c --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/ab_${c}_$v.json 2> gpurun_out/ab_${c}_$v.err
    python -c "import json;d=json.load(open('gpurun_out/ab_${c}_$v.json'));r=d['roofline'];print('$r $v $c', round(d['value'],1), 'TF/s | attn', round(r['achieved'],1), round(r['attn_ms_per_call']*1e3,1), 'us | issued', round(r.get('issued_tflops',0)), '| sel+plan', round(d['roofline_select']['select_plan_ms_per_call']*1e3,1), 'us | err', d['device_errors'])" || tail -n 5 gpurun_out/ab_${c}_$v.err
  done
done
done
