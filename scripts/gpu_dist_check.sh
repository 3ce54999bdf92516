# functional check of the multi-rank bench flow on one GPU (gloo, LF_BENCH_DIST_CHECK): head
# shards at N = 2 and 3 (c2: 6 / 4 heads per rank), replicas at N = 5; plus the N = 1 c2 line
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
for n in 2 3 5; do
  LF_BENCH_DIST_CHECK=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2951$n bench.py --gpus $n --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/dist_$n.json 2> gpurun_out/dist_$n.err
  echo "n=$n rc=$?"; tail -c 600 gpurun_out/dist_$n.json; echo; grep -i "error\|Traceback" gpurun_out/dist_$n.err | head -5
done
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/n1_c2.json 2> gpurun_out/n1_c2.err
python -c "import json;d=json.load(open('gpurun_out/n1_c2.json'));print('n1 c2', round(d['value'],1), d['step_order'][:6], 'e2e', round(d['e2e']['value']), round(d['e2e']['ms_per_chunk'],3))"
