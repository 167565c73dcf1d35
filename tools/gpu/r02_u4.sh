python -c "import __graft_entry__ as g; g.build()" || exit 1
mkdir -p gpurun_out
for r in 1 2; do for lib in libcdms libcdms_u4; do for c in c5 c3 c4; do
if [ $c = c5 ]; then PP="--particles 4000000"; else PP=""; fi
CDMS_LIB=paper_2604_19723_b200/$lib.so timeout 600 python bench.py --config $c $PP --steps 10 --no-cpu-baseline --no-extras > gpurun_out/r02_u4.json 2>gpurun_out/r02_u4.err
python -c "import json;d=json.load(open('gpurun_out/r02_u4.json'));print('$lib $c', round(d['ms_per_step'],3), d['kernel_ms_per_step'])"
done; done; done
CDMS_LIB=paper_2604_19723_b200/libcdms_u4.so timeout 900 python -m pytest tests/test_k1t_terms_gpu.py tests/test_parity_gpu.py -q -m gpu 2>&1 | tail -1
