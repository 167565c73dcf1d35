python -c "import __graft_entry__ as g; g.build()" || exit 1
mkdir -p gpurun_out
M=sm__inst_executed_pipe_fma.sum,sm__inst_executed_pipe_xu.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed,sm__inst_issued.avg.pct_of_peak_sustained_active
timeout 600 ncu --metrics $M -k regex:"tay_|assemble|dn_table" --csv --log-file gpurun_out/r02_fin_pipe_c5.csv python tools/run_step.py c5 600000 --steps 1 > gpurun_out/r02_fin2_n1.log 2>&1; echo ncu1 rc=$?
timeout 600 ncu --metrics $M -k regex:"tay_|assemble|dn_table" --csv --log-file gpurun_out/r02_fin_pipe_c3.csv python tools/run_step.py c3 1000000 --steps 1 > gpurun_out/r02_fin2_n2.log 2>&1; echo ncu2 rc=$?
timeout 600 ncu --metrics $M -k regex:"tay_|assemble" --csv --log-file gpurun_out/r02_fin_pipe_c2.csv python tools/run_step.py c2 100000 --steps 1 > gpurun_out/r02_fin2_n3.log 2>&1; echo ncu3 rc=$?
timeout 600 ncu --metrics $M -k regex:"tay_|assemble|dn_table" --csv --log-file gpurun_out/r02_fin_pipe_c4.csv python tools/run_step.py c4 1000000 --steps 1 > gpurun_out/r02_fin2_n4.log 2>&1; echo ncu4 rc=$?
timeout 900 ncu --set full --import-source on -k regex:"tay_gram|tay_corr|assemble" -c 3 -o gpurun_out/r02_fin_k1t_c5 python tools/run_step.py c5 600000 --steps 1 > gpurun_out/r02_fin2_n5.log 2>&1; echo ncu5 rc=$?
