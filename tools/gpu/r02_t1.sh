python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests/test_multirank_gpu.py tests/test_parity_gpu.py -x -q -m gpu 2>&1 | tail -30
