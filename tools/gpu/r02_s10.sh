python -c "import __graft_entry__ as g; g.build()" || exit 1
mkdir -p gpurun_out
timeout 900 python bench.py --mode slam --config exp1 --particles 30000 --steps 20 > gpurun_out/r02_slam_bench_exp1_p3e4.json 2>gpurun_out/r02_s10.err; python -c "import json;d=json.load(open('gpurun_out/r02_slam_bench_exp1_p3e4.json'));print(d['ms_per_step'], d['value'], d['vs_baseline'], d.get('cpu_baseline'))"
