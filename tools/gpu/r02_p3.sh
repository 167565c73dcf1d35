python -c "import __graft_entry__ as g; g.build()" || exit 1
mkdir -p gpurun_out
for lib in libcdms libcdms_p3m4 libcdms_p3m3; do
CDMS_LIB=paper_2604_19723_b200/$lib.so timeout 600 python bench.py --config c5 --particles 4000000 --steps 10 --no-cpu-baseline --no-extras > gpurun_out/r02_p3.json 2>gpurun_out/r02_p3.err
python -c "import json;d=json.load(open('gpurun_out/r02_p3.json'));print('$lib c5', round(d['ms_per_step'],3), d['kernel_ms_per_step'])"
done
