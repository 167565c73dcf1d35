python -c "import __graft_entry__ as g; g.build()" || exit 1
mkdir -p gpurun_out
PARITY_REPORT=gpurun_out/r02_fin3_parity.json timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
timeout 1200 python bench.py > gpurun_out/r02_fin3_bench_c5.json 2>gpurun_out/r02_fin3.err; python -c "import json;d=json.load(open('gpurun_out/r02_fin3_bench_c5.json'));print('c5', round(d['ms_per_step'],3), d['value'], d['roofline']['frac'], d['kernel_ms_per_step'])"
for c in c2 c3 c4; do
timeout 600 python bench.py --config $c --steps 20 --no-extras > gpurun_out/r02_fin3_bench_$c.json 2>>gpurun_out/r02_fin3.err
python -c "import json;d=json.load(open('gpurun_out/r02_fin3_bench_$c.json'));print('$c', round(d['ms_per_step'],3), d['value'], d['roofline']['frac'], d['kernel_ms_per_step'])"
done
M=sm__inst_executed_pipe_fma.sum,sm__inst_executed_pipe_xu.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
timeout 600 ncu --metrics $M -k regex:"tay_|assemble|dn_table" --csv --log-file gpurun_out/r02_fin3_pipe_c5.csv python tools/run_step.py c5 600000 --steps 1 > /dev/null 2>&1; echo ncu1 rc=$?
timeout 600 ncu --metrics $M -k regex:"tay_|assemble|dn_table" --csv --log-file gpurun_out/r02_fin3_pipe_c3.csv python tools/run_step.py c3 1000000 --steps 1 > /dev/null 2>&1; echo ncu2 rc=$?
timeout 600 ncu --metrics $M -k regex:"tay_|assemble|dn_table" --csv --log-file gpurun_out/r02_fin3_pipe_c2.csv python tools/run_step.py c2 100000 --steps 1 > /dev/null 2>&1; echo ncu3 rc=$?
timeout 600 ncu --metrics $M -k regex:"tay_|assemble|dn_table" --csv --log-file gpurun_out/r02_fin3_pipe_c4.csv python tools/run_step.py c4 1000000 --steps 1 > /dev/null 2>&1; echo ncu4 rc=$?
timeout 900 ncu --set full --import-source on -k regex:"tay_gram" -c 1 -o gpurun_out/r02_fin3_gram_c5 python tools/run_step.py c5 600000 --steps 1 > /dev/null 2>&1; echo ncu5 rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r02_fin3_launches_c5.csv python bench.py --particles 2000000 --steps 2 --warmup 3 --no-cpu-baseline --no-extras > /dev/null 2>&1; echo ncu6 rc=$?
