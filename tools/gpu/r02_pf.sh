python -c "import __graft_entry__ as g; g.build()" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_pf_gpu.py tests/test_slam_step_gpu.py tests/test_slam_gpu.py -q -m gpu 2>&1 | tail -2
timeout 900 python bench.py --mode slam --config exp1 --particles 1000000 --no-cpu-baseline > gpurun_out/r02_pf_slam.json 2>gpurun_out/r02_pf.err; python -c "import json;d=json.loads(open('gpurun_out/r02_pf_slam.json').read().strip().splitlines()[-1]);print('slam 1e6', d['ms_per_step'])"
timeout 900 python bench.py --mode pf --config c3 --no-cpu-baseline > gpurun_out/r02_pf_f1.json 2>>gpurun_out/r02_pf.err; python -c "import json;d=json.loads(open('gpurun_out/r02_pf_f1.json').read().strip().splitlines()[-1]);print('f1 c3', d['ms_per_step'])"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_pf_launches.csv python bench.py --mode slam --config exp1 --particles 1000000 --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo ncu rc=$?
