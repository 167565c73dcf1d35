python -c "import __graft_entry__ as g; g.build()" || exit 1
mkdir -p gpurun_out
for L in 0 1; do for c in c5 c3; do
if [ $c = c5 ]; then PP="--particles 4000000"; else PP=""; fi
CDMS_LOCALITY=$L timeout 600 python bench.py --config $c $PP --steps 10 --no-cpu-baseline --no-extras > gpurun_out/r02_ln.json 2>gpurun_out/r02_ln.err
python -c "import json;d=json.load(open('gpurun_out/r02_ln.json'));print('loc=$L $c', round(d['ms_per_step'],3), d['kernel_ms_per_step'])"
done; done
