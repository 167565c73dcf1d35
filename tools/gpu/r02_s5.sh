python -c "import __graft_entry__ as g; g.build()" || exit 1
mkdir -p gpurun_out
PARITY_REPORT=gpurun_out/r02_s5_parity.json timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
timeout 900 python bench.py --mode slam --config exp1 --particles 1000000 --steps 10 --warmup 3 > gpurun_out/r02_slam_bench_exp1_p1e6.json 2>gpurun_out/r02_s5.err; cat gpurun_out/r02_slam_bench_exp1_p1e6.json | cut -c1-300
timeout 900 python bench.py --mode slam --config exp1 --particles 100000 --steps 10 --warmup 3 > gpurun_out/r02_slam_bench_exp1_p1e5.json 2>>gpurun_out/r02_s5.err; cat gpurun_out/r02_slam_bench_exp1_p1e5.json | cut -c1-300
timeout 900 python bench.py --mode pf --config c3 --particles 1000000 --steps 10 --no-cpu-baseline > gpurun_out/r02_f1_bench_c3.json 2>>gpurun_out/r02_s5.err; cat gpurun_out/r02_f1_bench_c3.json | cut -c1-300
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_slam_launches.csv python bench.py --mode slam --config exp1 --particles 1000000 --steps 2 --warmup 3 > /dev/null 2>&1; echo ncu rc=$?
