# one ncu --set full capture of the attention kernel (config $NCU_CONFIG, env passed through)
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_fwd -s 1 -c 1 -o gpurun_out/${NCU_OUT:-attn_prof} python bench.py --profile-launch --no-cpu-baseline --config ${NCU_CONFIG:-c2} > gpurun_out/ncu_attn.log 2>&1
tail -n 3 gpurun_out/ncu_attn.log
