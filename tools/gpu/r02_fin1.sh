python -c "import __graft_entry__ as g; g.build()" || exit 1
mkdir -p gpurun_out
timeout 1200 python bench.py > gpurun_out/r02_fin_bench_c5.json 2>gpurun_out/r02_fin.err; cat gpurun_out/r02_fin_bench_c5.json | cut -c1-400
for c in c2 c3 c4; do
timeout 600 python bench.py --config $c --steps 20 --no-extras > gpurun_out/r02_fin_bench_$c.json 2>>gpurun_out/r02_fin.err
python -c "import json;d=json.load(open('gpurun_out/r02_fin_bench_$c.json'));print('$c', round(d['ms_per_step'],3), d['value'], d['roofline']['frac'], d['kernel_ms_per_step'])"
done
timeout 600 python bench.py --config c4 --wavefront planar_nb --steps 20 --no-extras > gpurun_out/r02_fin_bench_c4nb.json 2>>gpurun_out/r02_fin.err
python -c "import json;d=json.load(open('gpurun_out/r02_fin_bench_c4nb.json'));print('c4nb', round(d['ms_per_step'],3), d['value'], d['roofline'])"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r02_fin_launches_c5.csv python bench.py --particles 2000000 --steps 2 --warmup 3 --no-cpu-baseline --no-extras > /dev/null 2>&1; echo ncu1 rc=$?
