python -c "import __graft_entry__ as g; g.build()" || exit 1
mkdir -p gpurun_out
(cd tools/microbench && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o sincos_range sincos_range.cu && ./sincos_range) | tee gpurun_out/r02_sincos_range.txt
for c in c5 c3 c2 c4; do
if [ $c = c5 ]; then PP="--particles 4000000"; else PP=""; fi
timeout 600 python bench.py --config $c $PP --steps 10 --no-cpu-baseline --no-extras > gpurun_out/r02_cr.json 2>gpurun_out/r02_cr.err
python -c "import json;d=json.load(open('gpurun_out/r02_cr.json'));print('$c', round(d['ms_per_step'],3), d['kernel_ms_per_step'])"
done
timeout 900 python -m pytest tests -q -m gpu 2>&1 | tail -3
