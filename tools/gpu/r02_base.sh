set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python bench.py --config c5 --particles 16000000 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02_base_c5_16M.json 2> gpurun_out/r02_base_c5.err
timeout 600 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02_base_c3.json 2> gpurun_out/r02_base_c3.err
timeout 600 python bench.py --config c5 --particles 16000000 --precision fp64 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r02_base_c5_fp64.json 2> gpurun_out/r02_base_c5_fp64.err
tail -c 600 gpurun_out/*.json
