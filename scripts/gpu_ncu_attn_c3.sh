python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_fwd -s 1 -c 1 -o gpurun_out/attn_c3 -f python bench.py --profile-launch --no-cpu-baseline --config c3 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_fwd -s 1 -c 1 -o gpurun_out/attn_c5s70 -f python bench.py --profile-launch --no-cpu-baseline --config c5_s70 > /dev/null 2>&1
ls gpurun_out/*.ncu-rep
