# bench lines with the updated pipe counts (profiles/pipe_inst.json from r02_g3_pipe_*.csv)
python -c "import __graft_entry__ as g; g.build()" || exit 1
mkdir -p gpurun_out
timeout 1200 python bench.py > gpurun_out/r02_g4_bench_c5.json 2>gpurun_out/r02_g4.err; python -c "import json;d=json.load(open('gpurun_out/r02_g4_bench_c5.json'));print('c5', round(d['ms_per_step'],3), d['value'], d['roofline']['frac'], d['roofline'].get('limiter',{}).get('pipe'), d['kernel_ms_per_step'], d['e2e']['value'])"
for c in c2 c3 c4; do
timeout 600 python bench.py --config $c --steps 20 --no-extras > gpurun_out/r02_g4_bench_$c.json 2>>gpurun_out/r02_g4.err
python -c "import json;d=json.load(open('gpurun_out/r02_g4_bench_$c.json'));print('$c', round(d['ms_per_step'],3), d['value'], d['roofline']['frac'], d['kernel_ms_per_step'])"
done
timeout 900 python bench.py --mode pf --config c3 > gpurun_out/r02_g4_f1_c3.json 2>>gpurun_out/r02_g4.err; tail -c 300 gpurun_out/r02_g4_f1_c3.json
