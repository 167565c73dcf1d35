python -c "import __graft_entry__ as g; g.build()" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_slam_gpu.py tests/test_slam_step_gpu.py -q -m gpu -x 2>&1 | tail -3
timeout 900 python bench.py --mode slam --config exp1 --particles 1000000 --steps 10 --warmup 3 > gpurun_out/r02_slam_bench_exp1_p1e6.json 2>gpurun_out/r02_s6.err; cat gpurun_out/r02_slam_bench_exp1_p1e6.json | cut -c1-300
