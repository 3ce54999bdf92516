python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
LF_QTILE=paired timeout 600 ncu --set full --import-source on --clock-control none -k regex:pair_qblocks -s 2 -c 1 -o gpurun_out/pair_c3 -f python bench.py --config c3 --steps 2 --warmup 1 --no-cpu-baseline --profile-launch > gpurun_out/ncu_pair.log 2>&1
ncu -i gpurun_out/pair_c3.ncu-rep --page details --csv > gpurun_out/pair_details.csv 2>&1
ncu -i gpurun_out/pair_c3.ncu-rep --page source --csv > gpurun_out/pair_source.csv 2>&1
LF_QTILE=paired timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launch_pair_c3.csv python bench.py --config c3 --steps 2 --warmup 1 --no-cpu-baseline --profile-launch > /dev/null 2>&1
tail -2 gpurun_out/ncu_pair.log
