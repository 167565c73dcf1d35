python -c "import __graft_entry__ as g; g.build()" || exit 1
mkdir -p gpurun_out
PARITY_REPORT=gpurun_out/r02_dn_parity.json timeout 900 python -m pytest tests/test_k1t_terms_gpu.py tests/test_parity_gpu.py -q -m gpu -x 2>&1 | tail -2
for lib in libcdms libcdms_d64 libcdms_deg7; do for c in c5 c3 c2 c4; do
if [ $c = c5 ]; then PP="--particles 4000000"; else PP=""; fi
for tab in 1 2; do
if [ $tab = 2 ] && { [ $c = c5 ] || [ $c = c3 ]; }; then continue; fi
CDMS_GRAM_TAB=$tab CDMS_LIB=paper_2604_19723_b200/$lib.so timeout 600 python bench.py --config $c $PP --steps 10 --no-cpu-baseline --no-extras > gpurun_out/r02_dn.json 2>gpurun_out/r02_dn.err
python -c "import json;d=json.load(open('gpurun_out/r02_dn.json'));print('$lib tab=$tab $c', round(d['ms_per_step'],3), d['kernel_ms_per_step'])"
done; done; done
