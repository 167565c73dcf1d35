python -c "import __graft_entry__ as g; g.build()" || exit 1
mkdir -p gpurun_out
for P in 1000000 100000 30000; do
timeout 900 python bench.py --mode slam --config exp1 --particles $P > gpurun_out/r02_f4_slam_$P.json 2>>gpurun_out/r02_f4.err; python -c "import json;d=json.loads(open('gpurun_out/r02_f4_slam_$P.json').read().strip().splitlines()[-1]);print('slam $P', d['ms_per_step'], d['value'], d.get('vs_baseline'))"
done
timeout 900 python bench.py --mode pf --config c3 > gpurun_out/r02_f4_f1_c3.json 2>>gpurun_out/r02_f4.err; python -c "import json;d=json.loads(open('gpurun_out/r02_f4_f1_c3.json').read().strip().splitlines()[-1]);print('f1 c3', d['ms_per_step'], d['value'])"
timeout 900 python bench.py --mode pf --config c2 > gpurun_out/r02_f4_f1_c2.json 2>>gpurun_out/r02_f4.err; python -c "import json;d=json.loads(open('gpurun_out/r02_f4_f1_c2.json').read().strip().splitlines()[-1]);print('f1 c2', d['ms_per_step'], d['value'])"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_f4_launches.csv python bench.py --mode slam --config exp1 --particles 1000000 --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo ncu rc=$?
