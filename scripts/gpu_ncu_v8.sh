python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
for v in 7 8; do
LF_TILE_VER=$v timeout 600 ncu --set full --import-source on --clock-control none -k regex:attn_fwd -s 2 -c 1 -o gpurun_out/attn_v${v}_c5d -f python bench.py --config c5_dense --steps 2 --warmup 1 --no-cpu-baseline --profile-launch > gpurun_out/ncu_v$v.log 2>&1
ncu -i gpurun_out/attn_v${v}_c5d.ncu-rep --page details --csv > gpurun_out/attn_v${v}_details.csv 2>&1
ncu -i gpurun_out/attn_v${v}_c5d.ncu-rep --page source --csv > gpurun_out/attn_v${v}_source.csv 2>&1
ncu -i gpurun_out/attn_v${v}_c5d.ncu-rep --page raw --csv > gpurun_out/attn_v${v}_raw.csv 2>&1
tail -2 gpurun_out/ncu_v$v.log
done
