# final measurement after the Gram, assembly and carrier changes: parity, benches, pipe counts, warm ncu, launch list
python -c "import __graft_entry__ as g; g.build()" || exit 1
mkdir -p gpurun_out
PARITY_REPORT=gpurun_out/r02_g11_parity.json timeout 1500 python -m pytest tests -q -m gpu 2>&1 | tail -2
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1200 python bench.py > gpurun_out/r02_g11_bench_c5.json 2>gpurun_out/r02_g11.err; python -c "import json;d=json.load(open('gpurun_out/r02_g11_bench_c5.json'));print('c5', round(d['ms_per_step'],3), d['value'], d['roofline']['frac'], d['kernel_ms_per_step'])"
for c in c2 c3 c4; do
timeout 600 python bench.py --config $c --steps 20 --no-extras > gpurun_out/r02_g11_bench_$c.json 2>>gpurun_out/r02_g11.err
python -c "import json;d=json.load(open('gpurun_out/r02_g11_bench_$c.json'));print('$c', round(d['ms_per_step'],3), d['value'], d['roofline']['frac'], d['kernel_ms_per_step'])"
done
M=sm__inst_executed_pipe_fma.sum,sm__inst_executed_pipe_xu.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
for c in "c5 600000" "c3 1000000" "c2 100000" "c4 1000000"; do set -- $c
timeout 600 ncu --metrics $M -k regex:"tay_|assemble|dn_table" --csv --log-file gpurun_out/r02_g11_pipe_$1.csv python tools/run_step.py $1 $2 --steps 1 > /dev/null 2>&1; echo ncu $1 rc=$?
done
timeout 900 ncu --set full --cache-control none --clock-control none -k regex:"tay_corr_kernel" -s 2 -c 1 -o gpurun_out/r02_g11_warm python tools/run_step.py c5 600000 --steps 3 > gpurun_out/r02_g11_warm.log 2>&1; echo ncu warm rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_g11_launches_c5.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r02_g11_ncu.log 2>&1; echo ncu launches rc=$?
timeout 900 python bench.py --mode slam --config exp1 --particles 1000000 > gpurun_out/r02_g11_slam_p1e6.json 2>>gpurun_out/r02_g11.err; tail -c 400 gpurun_out/r02_g11_slam_p1e6.json
timeout 900 python bench.py --mode slam --config exp1 --particles 30000 > gpurun_out/r02_g11_slam_p3e4.json 2>>gpurun_out/r02_g11.err; tail -c 300 gpurun_out/r02_g11_slam_p3e4.json
timeout 900 python bench.py --mode pf --config c3 > gpurun_out/r02_g11_f1_c3.json 2>>gpurun_out/r02_g11.err; tail -c 300 gpurun_out/r02_g11_f1_c3.json
