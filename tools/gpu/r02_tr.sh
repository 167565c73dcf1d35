python -c "import __graft_entry__ as g; g.build()" || exit 1
mkdir -p gpurun_out
timeout 900 python tools/slam_run.py --init map --particles 1000000 --steps 60 --out gpurun_out/r02_slam_map_p1e6.jsonl > /dev/null 2>gpurun_out/r02_tr.err; tail -1 gpurun_out/r02_slam_map_p1e6.jsonl
timeout 900 python tools/slam_run.py --init map --particles 100000 --steps 60 --out gpurun_out/r02_slam_map_p1e5.jsonl > /dev/null 2>>gpurun_out/r02_tr.err; tail -1 gpurun_out/r02_slam_map_p1e5.jsonl
timeout 900 python tools/slam_run.py --init scratch --particles 1000000 --steps 60 --out gpurun_out/r02_slam_scratch_p1e6.jsonl > /dev/null 2>>gpurun_out/r02_tr.err; tail -1 gpurun_out/r02_slam_scratch_p1e6.jsonl
