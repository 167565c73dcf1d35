python -c "import __graft_entry__ as g; g.build()" || exit 1
mkdir -p gpurun_out
for lib in libcdms libcdms_tb8 libcdms_tb32; do
CDMS_LIB=paper_2604_19723_b200/$lib.so timeout 900 python bench.py --steps 10 --no-cpu-baseline --no-extras > gpurun_out/r02_tb.json 2>gpurun_out/r02_tb.err
python -c "import json;d=json.load(open('gpurun_out/r02_tb.json'));print('$lib c5', round(d['ms_per_step'],3), d['kernel_ms_per_step'])"
done
