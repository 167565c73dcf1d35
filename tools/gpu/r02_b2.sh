python -c "import __graft_entry__ as g; g.build()" || exit 1
mkdir -p gpurun_out
for c in c3 c2; do
timeout 600 python bench.py --mode pf --config $c --steps 10 --cpu-seconds 6 > gpurun_out/r02_b2_pf_$c.json 2>gpurun_out/r02_b2_pf_$c.err; echo pf $c rc=$?
tail -c 1500 gpurun_out/r02_b2_pf_$c.json
done
M=sm__inst_executed_pipe_fma.sum,sm__inst_executed_pipe_xu.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
timeout 600 ncu --metrics $M -k regex:"tay_|assemble" --csv --log-file gpurun_out/r02_b2_pipe_c5.csv python tools/run_step.py c5 600000 --steps 1 > gpurun_out/r02_b2_ncu1.log 2>&1; echo ncu1 rc=$?
timeout 600 ncu --metrics $M -k regex:"tay_|assemble" --csv --log-file gpurun_out/r02_b2_pipe_c3.csv python tools/run_step.py c3 1000000 --steps 1 > gpurun_out/r02_b2_ncu2.log 2>&1; echo ncu2 rc=$?
timeout 900 ncu --set full --import-source on -k regex:"tay_gram|tay_corr" -c 2 -o gpurun_out/r02_b2_k1t_c5 python tools/run_step.py c5 600000 --steps 1 > gpurun_out/r02_b2_ncu3.log 2>&1; echo ncu3 rc=$?
