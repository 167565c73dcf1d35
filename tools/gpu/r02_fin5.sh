python -c "import __graft_entry__ as g; g.build()" || exit 1
mkdir -p gpurun_out
M=sm__inst_executed_pipe_fma.sum,sm__inst_executed_pipe_xu.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
for c in "c5 600000" "c3 1000000" "c2 100000" "c4 1000000"; do set -- $c
timeout 600 ncu --metrics $M -k regex:"tay_|assemble|dn_table" --csv --log-file gpurun_out/r02_fin5_pipe_$1.csv python tools/run_step.py $1 $2 --steps 1 > /dev/null 2>&1; echo ncu $1 rc=$?
done
timeout 900 ncu --set full --import-source on -k regex:"tay_gram|tay_corr" -c 2 -o gpurun_out/r02_fin5_k1t_c5 python tools/run_step.py c5 600000 --steps 1 > /dev/null 2>&1; echo ncu full rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r02_fin5_launches_c5.csv python bench.py --particles 2000000 --steps 2 --warmup 3 --no-cpu-baseline --no-extras > /dev/null 2>&1; echo ncu launches rc=$?
