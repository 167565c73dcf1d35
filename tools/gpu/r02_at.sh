python -c "import __graft_entry__ as g; g.build()" || exit 1
mkdir -p gpurun_out
for lib in libcdms libcdms_a64 libcdms_a256; do for c in c5 c3; do
if [ $c = c5 ]; then PP="--particles 4000000"; else PP=""; fi
CDMS_LIB=paper_2604_19723_b200/$lib.so timeout 600 python bench.py --config $c $PP --steps 10 --no-cpu-baseline --no-extras > gpurun_out/r02_at.json 2>gpurun_out/r02_at.err
python -c "import json;d=json.load(open('gpurun_out/r02_at.json'));print('$lib $c', round(d['ms_per_step'],3), d['kernel_ms_per_step'])"
done; done
