python -c "import __graft_entry__ as g; g.build()" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_k1t_terms_gpu.py "tests/test_parity_gpu.py::test_loglik_ragged_shapes" -q -m gpu -p no:cacheprovider 2>&1 | tail -40
PARITY_REPORT=gpurun_out/r02_t2_parity.json timeout 900 python -m pytest tests/test_k1t_terms_gpu.py -q -m gpu 2>&1 | tail -2
timeout 900 ncu --set full --import-source on -k regex:"tay_gram|tay_corr" --launch-skip 2 -c 2 -o gpurun_out/r02_t2_k1t_c5 python tools/run_step.py c5 2000000 --steps 1 > gpurun_out/r02_t2_ncu.log 2>&1; echo ncu rc=$?
