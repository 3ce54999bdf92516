# bench + ncu evidence on one B200 (run via gpurun)
set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 600 python bench.py --steps 50 --warmup 5 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
for c in c3 c4 c5_dense c5_s50 c5_s70 c5_s85; do
  timeout 300 python bench.py --config $c --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_c2.json 2> gpurun_out/bench_ref_c2.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python bench.py --profile-launch --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_fwd -s 2 -c 1 -o gpurun_out/attn_c2 python bench.py --profile-launch --no-cpu-baseline > gpurun_out/ncu_attn.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_fwd -s 2 -c 1 -o gpurun_out/attn_c5_dense python bench.py --profile-launch --no-cpu-baseline --config c5_dense > gpurun_out/ncu_attn5.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pool_frames -s 2 -c 1 -o gpurun_out/pool_c2 python bench.py --profile-launch --no-cpu-baseline > gpurun_out/ncu_pool.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:select_cta -s 2 -c 1 -o gpurun_out/select_c5_dense python bench.py --profile-launch --no-cpu-baseline --config c5_dense > gpurun_out/ncu_select.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:select_cta -s 2 -c 1 -o gpurun_out/select_c3 python bench.py --profile-launch --no-cpu-baseline --config c3 > gpurun_out/ncu_select3.log 2>&1
tail -n 3 gpurun_out/*.err
