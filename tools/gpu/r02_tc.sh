python -c "import __graft_entry__ as g; g.build()" || exit 1
mkdir -p gpurun_out
for c in c5 c3 c2 c4; do
if [ $c = c5 ]; then PP="--particles 4000000"; else PP=""; fi
timeout 600 python bench.py --config $c $PP --steps 10 --no-cpu-baseline --no-extras > gpurun_out/r02_tc.json 2>gpurun_out/r02_tc.err
python -c "import json;d=json.load(open('gpurun_out/r02_tc.json'));print('$c', round(d['ms_per_step'],3), d['kernel_ms_per_step'])"
done
timeout 1200 python -m pytest tests -q -m gpu 2>&1 | tail -1
