python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_rollout.py tests/test_gpu_paired.py tests/test_gpu_select_plan.py -m gpu -x -q 2>&1 | tail -2
bash scripts/gpu_timeline.sh
head -4 gpurun_out/timeline_c2.csv
