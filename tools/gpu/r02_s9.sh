python -c "import __graft_entry__ as g; g.build()" || exit 1
mkdir -p gpurun_out
timeout 900 python tools/slam_run.py --init scratch --particles 4000000 --steps 60 --out gpurun_out/r02_slam_scratch_p4e6.jsonl 2>&1 | tail -1
timeout 900 python tools/slam_run.py --init map --particles 1000000 --steps 60 --out gpurun_out/r02_slam_map_p1e6.jsonl 2>&1 | tail -1
