python -c "import __graft_entry__ as g; g.build()" || exit 1
mkdir -p gpurun_out
PARITY_REPORT=gpurun_out/r02_fin8_parity.json timeout 1500 python -m pytest tests -q -m gpu 2>&1 | tail -2
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
M=sm__inst_executed_pipe_fma.sum,sm__inst_executed_pipe_xu.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
for c in "c5 600000" "c3 1000000" "c2 100000" "c4 1000000"; do set -- $c
timeout 600 ncu --metrics $M -k regex:"tay_|assemble|dn_table" --csv --log-file gpurun_out/r02_fin8_pipe_$1.csv python tools/run_step.py $1 $2 --steps 1 > /dev/null 2>&1; echo ncu $1 rc=$?
done
