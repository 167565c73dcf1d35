python -c "import __graft_entry__ as g; g.build()" || exit 1
mkdir -p gpurun_out
PARITY_REPORT=gpurun_out/r02_t8_parity.json timeout 1500 python -m pytest tests/test_pf_gpu.py -q -m gpu 2>&1 | tail -3
