python -c "import __graft_entry__ as g; g.build()" || exit 1
mkdir -p gpurun_out
for r in 1 2; do for lib in libcdms libcdms_un8 libcdms_un16; do for c in c5 c3; do
if [ $c = c5 ]; then PP="--particles 4000000"; else PP=""; fi
CDMS_LIB=paper_2604_19723_b200/$lib.so timeout 600 python bench.py --config $c $PP --steps 10 --no-cpu-baseline --no-extras > gpurun_out/r02_un.json 2>gpurun_out/r02_un.err
python -c "import json;d=json.load(open('gpurun_out/r02_un.json'));print('$lib $c', round(d['ms_per_step'],3), d['kernel_ms_per_step'])"
done; done; done
