python -c "import __graft_entry__ as g; g.build()" || exit 1
mkdir -p gpurun_out
timeout 1500 python tools/slam_run.py --init roi --particles 16000000 --steps 80 --out gpurun_out/r02_slam_roi_p16e6.jsonl 2>&1 | tail -1
