python -c "import __graft_entry__ as g; g.build()" || exit 1
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/r02_b1_c5.json 2> gpurun_out/r02_b1_c5.err; echo bench rc=$?
tail -c 2500 gpurun_out/r02_b1_c5.json
M=sm__inst_executed_pipe_fma.sum,sm__inst_executed_pipe_xu.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
timeout 600 ncu --metrics $M -k regex:"tay_|assemble" --launch-skip 4 -c 4 --csv --log-file gpurun_out/r02_b1_pipe_c5.csv python tools/run_step.py c5 2000000 > gpurun_out/r02_b1_ncu.log 2>&1; echo ncu rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/r02_b1_launches_c5.csv python tools/run_step.py c5 2000000 > /dev/null 2>&1; echo ncu2 rc=$?
