# bench lines with the pipe counts of r02_g11 (profiles/pipe_inst.json)
python -c "import __graft_entry__ as g; g.build()" || exit 1
mkdir -p gpurun_out
timeout 1200 python bench.py > gpurun_out/r02_g12_bench_c5.json 2>gpurun_out/r02_g12.err; python -c "import json;d=json.load(open('gpurun_out/r02_g12_bench_c5.json'));print('c5', round(d['ms_per_step'],3), d['value'], d['roofline']['frac'], d['roofline']['kernel'], d['kernel_ms_per_step'], d['e2e']['value'])"
for c in c2 c3 c4; do
timeout 600 python bench.py --config $c --steps 20 --no-extras > gpurun_out/r02_g12_bench_$c.json 2>>gpurun_out/r02_g12.err
python -c "import json;d=json.load(open('gpurun_out/r02_g12_bench_$c.json'));print('$c', round(d['ms_per_step'],3), d['value'], d['roofline']['frac'], d['roofline']['kernel'], d['kernel_ms_per_step'])"
done
timeout 900 python bench.py --config c4 --wavefront planar_nb --steps 20 --no-extras > gpurun_out/r02_g12_bench_c4nb.json 2>>gpurun_out/r02_g12.err; python -c "import json;d=json.load(open('gpurun_out/r02_g12_bench_c4nb.json'));print('c4nb', round(d['ms_per_step'],3), d['value'], d['kernel_ms_per_step'])"
