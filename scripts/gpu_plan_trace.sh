python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_select_plan.py tests/test_gpu_paired.py tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -2
PYTHONPATH=. timeout 300 python scripts/sel_micro.py plan
LF_NVCC_FLAGS="-DLF_PAIR_TRACE" python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
PYTHONPATH=. timeout 300 python scripts/sel_micro.py plan 2>&1 | grep pair_trace | sort | uniq | head -8
