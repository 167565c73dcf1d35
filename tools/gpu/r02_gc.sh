python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests/test_parity_gpu.py -q -m gpu -k "graph_capture" 2>&1 | tail -15
