python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
PYTHONPATH=. timeout 300 python scripts/sel_micro.py
