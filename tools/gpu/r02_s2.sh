python -c "import __graft_entry__ as g; g.build()" || exit 1
mkdir -p gpurun_out
timeout 900 python tools/slam_run.py --particles 100000 --steps 40 --out gpurun_out/r02_slam_run_p1e5.jsonl 2>&1 | tail -45
