python -c "import __graft_entry__ as g; g.build()" || exit 1
mkdir -p gpurun_out
PARITY_REPORT=gpurun_out/r02_s3_parity.json timeout 900 python -m pytest tests/test_slam_step_gpu.py -q -m gpu -x 2>&1 | tail -3
for init in map scratch; do
timeout 900 python tools/slam_run.py --init $init --particles 100000 --steps 60 --out gpurun_out/r02_slam_${init}_p1e5.jsonl 2>&1 | tail -1
done
timeout 900 python tools/slam_run.py --init scratch --particles 1000000 --steps 60 --out gpurun_out/r02_slam_scratch_p1e6.jsonl 2>&1 | tail -1
