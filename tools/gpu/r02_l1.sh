python -c "import __graft_entry__ as g; g.build()" || exit 1
mkdir -p gpurun_out
for loc in 0 1; do for c in c5 c3; do
if [ $c = c5 ]; then PP="--particles 4000000"; else PP=""; fi
CDMS_LOCALITY=$loc timeout 600 python bench.py --config $c $PP --steps 10 --no-cpu-baseline --no-extras > gpurun_out/r02_l1.json 2>gpurun_out/r02_l1.err
python -c "import json;d=json.load(open('gpurun_out/r02_l1.json'));print('loc=$loc $c', round(d['ms_per_step'],3), d['kernel_ms_per_step'])"
done; done
