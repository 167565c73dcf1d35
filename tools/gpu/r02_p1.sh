python -c "import __graft_entry__ as g; g.build()" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_k1t_terms_gpu.py -q -m gpu -x -k "terms_parity" 2>&1 | tail -3
for c in c5 c3 c2; do
timeout 600 python bench.py --config $c --steps 10 --no-cpu-baseline --no-extras > gpurun_out/r02_p1_$c.json 2>gpurun_out/r02_p1_$c.err
python -c "import json;d=json.load(open('gpurun_out/r02_p1_$c.json'));print('$c', round(d['ms_per_step'],3), d['kernel_ms_per_step'])"
done
