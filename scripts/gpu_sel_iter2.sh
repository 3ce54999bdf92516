python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_select_plan.py tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -2
PYTHONPATH=. timeout 300 python scripts/sel_micro.py 2>&1 | grep -v "undecided"
bash scripts/gpu_sel_trace.sh
