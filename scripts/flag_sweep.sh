# rebuild the library per nvcc flag set and bench each (run via gpurun):
#   FLAGSETS="-DA=1 -DB=2|-DA=2" CONFIGS="c2 c5_dense" bash scripts/flag_sweep.sh
IFS='|' read -ra SETS <<< "${FLAGSETS:-}"
[ ${#SETS[@]} -eq 0 ] && SETS=("")
for fl in "${SETS[@]}"; do
  LF_NVCC_FLAGS="$fl" python -c "import __graft_entry__ as g; g.build()" > /dev/null || { echo "build failed: $fl"; continue; }
  tag=$(echo "$fl" | tr -d ' -' | tr '=' '_')
  for c in ${CONFIGS:-c2}; do
    timeout 300 python bench.py --config $c --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/fs_${c}_$tag.json 2> gpurun_out/fs_${c}_$tag.err
    python -c "import json;d=json.load(open('gpurun_out/fs_${c}_$tag.json'));r=d['roofline'];print('[$fl] $c', round(d['value'],1), 'TF/s | attn', round(r['achieved'],1), round(r['attn_ms_per_call']*1e3,1), 'us | issued', round(r.get('issued_tflops',0)), '| err', d['device_errors'])" || tail -n 5 gpurun_out/fs_${c}_$tag.err
  done
done
LF_NVCC_FLAGS= python -c "import __graft_entry__ as g; g.build()" > /dev/null
