python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
export PYTHONPATH=.
timeout 300 ncu --set full --clock-control none --import-source on -k regex:select_screen -s 2 -c 1 -o gpurun_out/sel1_c5_s70 -f python scripts/sel_micro.py c5_s70 1 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:select_screen -s 2 -c 1 -o gpurun_out/sel1_c3 -f python scripts/sel_micro.py c3 1 > /dev/null 2>&1
ls gpurun_out
