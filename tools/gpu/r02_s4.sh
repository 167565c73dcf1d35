python -c "import __graft_entry__ as g; g.build()" || exit 1
mkdir -p gpurun_out
timeout 900 python bench.py --mode slam --config exp1 --particles 1000000 --steps 10 --warmup 3 > gpurun_out/r02_slam_bench_exp1_p1e6.json 2>gpurun_out/r02_s4.err; tail -3 gpurun_out/r02_s4.err; cat gpurun_out/r02_slam_bench_exp1_p1e6.json
timeout 900 python bench.py --mode slam --config exp1 --particles 100000 --steps 10 --warmup 3 > gpurun_out/r02_slam_bench_exp1_p1e5.json 2>>gpurun_out/r02_s4.err; cat gpurun_out/r02_slam_bench_exp1_p1e5.json
timeout 600 nsys --version > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_slam_launches.csv python bench.py --mode slam --config exp1 --particles 1000000 --steps 2 --warmup 3 > /dev/null 2>&1; echo ncu rc=$?
