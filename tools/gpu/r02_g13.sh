# final bench lines (32 GiB terms budget: the c5 step in one likelihood batch) and the default command's launch list
python -c "import __graft_entry__ as g; g.build()" || exit 1
mkdir -p gpurun_out
timeout 1200 python bench.py > gpurun_out/r02_g13_bench_c5.json 2>gpurun_out/r02_g13.err; python -c "import json;d=json.load(open('gpurun_out/r02_g13_bench_c5.json'));print('c5', round(d['ms_per_step'],3), d['value'], d['roofline']['frac'], d['roofline']['kernel'], d['kernel_ms_per_step'], d['e2e']['value'], d['gpu_launches'])"
for c in c2 c3 c4; do
timeout 600 python bench.py --config $c --steps 20 --no-extras > gpurun_out/r02_g13_bench_$c.json 2>>gpurun_out/r02_g13.err
python -c "import json;d=json.load(open('gpurun_out/r02_g13_bench_$c.json'));print('$c', round(d['ms_per_step'],3), d['value'], d['roofline']['frac'], d['kernel_ms_per_step'])"
done
timeout 900 python bench.py --config c4 --wavefront planar_nb --steps 20 --no-extras > gpurun_out/r02_g13_bench_c4nb.json 2>>gpurun_out/r02_g13.err; python -c "import json;d=json.load(open('gpurun_out/r02_g13_bench_c4nb.json'));print('c4nb', round(d['ms_per_step'],3), d['value'])"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_g13_launches_c5.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r02_g13_ncu.log 2>&1; echo ncu launches rc=$?
timeout 900 python bench.py --mode slam --config exp1 --particles 1000000 > gpurun_out/r02_g13_slam_p1e6.json 2>>gpurun_out/r02_g13.err
timeout 900 python bench.py --mode slam --config exp1 --particles 30000 > gpurun_out/r02_g13_slam_p3e4.json 2>>gpurun_out/r02_g13.err
timeout 900 python bench.py --mode pf --config c3 > gpurun_out/r02_g13_f1_c3.json 2>>gpurun_out/r02_g13.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r02_g13_ref.json 2>>gpurun_out/r02_g13.err; echo ref rc=$?
