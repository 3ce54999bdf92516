LF_NVCC_FLAGS=-DLF_SEL_TRACE python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
export PYTHONPATH=.
for c in c2 c5_s70; do for H in 1 12; do echo "== $c H=$H"; timeout 120 python scripts/sel_micro.py $c $H | tail -3; done; done
