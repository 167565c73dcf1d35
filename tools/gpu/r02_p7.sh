python -c "import __graft_entry__ as g; g.build()" || exit 1
mkdir -p gpurun_out
PARITY_REPORT=gpurun_out/r02_p7_parity.json timeout 900 python -m pytest tests/test_k1t_terms_gpu.py -q -m gpu -x -k "terms_parity" 2>&1 | tail -2
for tab in 1 0; do for c in c5 c3 c2 c4; do
if [ $c = c5 ]; then PP="--particles 4000000"; else PP=""; fi
CDMS_GRAM_TAB=$tab timeout 600 python bench.py --config $c $PP --steps 10 --no-cpu-baseline --no-extras > gpurun_out/r02_p7.json 2>gpurun_out/r02_p7.err
python -c "import json;d=json.load(open('gpurun_out/r02_p7.json'));print('tab=$tab $c', round(d['ms_per_step'],3), d['kernel_ms_per_step'])"
done; done
