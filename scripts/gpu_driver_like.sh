# what the driver runs at round end (1 GPU): reference arm, our arm, --gpus 2 refusal
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/ref1.json 2> gpurun_out/ref1.err; echo ref rc=$?
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/n1.json 2> gpurun_out/n1.err; echo ours rc=$?
timeout 300 python bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/n2.json 2> gpurun_out/n2.err; echo "gpus2 rc=$? (expected 2)"; cat gpurun_out/n2.err | tail -2
python - <<'PY'
import json
r=json.load(open('gpurun_out/ref1.json')); o=json.load(open('gpurun_out/n1.json'))
print('ref', r['value'], r['cpu_baseline']['kind'], (r.get('port_framewise') or {}).get('value'))
print('ours', o['value'], 'e2e', o['e2e']['value'], 'stateless', o['stateless']['value'], 'attn frac', o['roofline']['frac'], 'stage frac', o['roofline_select']['frac'], 'pool frac', o['roofline_select']['pool_frac'])
print('cpu', o['cpu_baseline']['value'], o['cpu_baseline']['kind'], o['cpu_baseline'].get('port_framewise',{}).get('value'))
print('same config', r['config']==o['config'])
PY
