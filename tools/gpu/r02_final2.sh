python -c "import __graft_entry__ as g; g.build()" || exit 1
mkdir -p gpurun_out
PARITY_REPORT=gpurun_out/r02_final2_parity.json timeout 1500 python -m pytest tests -q -m gpu 2>&1 | tail -2
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1200 python bench.py > gpurun_out/r02_final2_bench.json 2>gpurun_out/r02_final2.err; python -c "import json;d=json.load(open('gpurun_out/r02_final2_bench.json'));print('c5', round(d['ms_per_step'],3), d['value'], d['roofline']['frac'], d['e2e']['value'], d['clocks'])"
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r02_final2_ref.json 2>>gpurun_out/r02_final2.err; tail -c 400 gpurun_out/r02_final2_ref.json
