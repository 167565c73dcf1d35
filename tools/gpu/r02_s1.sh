python -c "import __graft_entry__ as g; g.build()" || exit 1
mkdir -p gpurun_out
PARITY_REPORT=gpurun_out/r02_s1_parity.json timeout 900 python -m pytest tests/test_slam_step_gpu.py tests/test_pf_gpu.py -q -m gpu -x 2>&1 | tail -40
