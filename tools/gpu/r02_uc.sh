python -c "import __graft_entry__ as g; g.build()" || exit 1
mkdir -p gpurun_out
PARITY_REPORT=gpurun_out/r02_uc_parity.json timeout 1500 python -m pytest tests/test_k1t_terms_gpu.py tests/test_parity_gpu.py -q -m gpu -x 2>&1 | tail -2
for c in c5 c3 c4 c2; do
if [ $c = c5 ]; then PP="--particles 4000000"; else PP=""; fi
timeout 600 python bench.py --config $c $PP --steps 10 --no-cpu-baseline --no-extras > gpurun_out/r02_uc.json 2>gpurun_out/r02_uc.err
python -c "import json;d=json.load(open('gpurun_out/r02_uc.json'));print('$c', round(d['ms_per_step'],3), d['kernel_ms_per_step'])"
done
