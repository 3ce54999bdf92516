# ncu evidence after the block-aligned tiles / 4-group pooling change (run via gpurun, one GPU)
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python bench.py --profile-launch --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv python bench.py --profile-launch --no-cpu-baseline --config c3 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pool_frames -s 2 -c 1 -o gpurun_out/pool_c2 python bench.py --profile-launch --no-cpu-baseline > gpurun_out/ncu_pool.log 2>&1
LF_QTILE=blocks timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_fwd -s 1 -c 1 -o gpurun_out/attn_c3_blocks python bench.py --profile-launch --no-cpu-baseline --config c3 > gpurun_out/ncu_attn3.log 2>&1
LF_QTILE=rows timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_fwd -s 1 -c 1 -o gpurun_out/attn_c3_rows python bench.py --profile-launch --no-cpu-baseline --config c3 > gpurun_out/ncu_attn3r.log 2>&1
tail -n 2 gpurun_out/ncu_*.log
ls -la gpurun_out/*.ncu-rep
