python -c "import __graft_entry__ as g; g.build()" || exit 1
mkdir -p gpurun_out
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_c5_default.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extras > gpurun_out/r02_launch_bench.json 2>gpurun_out/r02_launch.err; echo ncu rc=$?
timeout 900 python bench.py --mode slam --config exp1 --particles 1000000 --steps 10 > gpurun_out/r02_fin7_slam_p1e6.json 2>>gpurun_out/r02_launch.err; python -c "import json;d=json.load(open('gpurun_out/r02_fin7_slam_p1e6.json'));print(d['ms_per_step'], d.get('cpu_baseline'))"
