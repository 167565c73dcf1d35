python -c "import __graft_entry__ as g; g.build()" || exit 1
mkdir -p gpurun_out
for loc in 0 1; do for c in c5 c3; do
if [ $c = c5 ]; then PP="--particles 4000000"; else PP=""; fi
CDMS_LOCALITY=$loc timeout 600 python bench.py --config $c $PP --steps 10 --no-cpu-baseline --no-extras > gpurun_out/r02_loc2.json 2>gpurun_out/r02_loc2.err
python -c "import json;d=json.load(open('gpurun_out/r02_loc2.json'));print('loc=$loc $c', round(d['ms_per_step'],3), d['kernel_ms_per_step'])"
done; done
M=l1tex__data_pipe_lsu_wavefronts.sum,smsp__inst_executed.sum,gpu__time_duration.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum
for loc in 0 1; do
CDMS_LOCALITY=$loc timeout 600 ncu --metrics $M -k regex:"tay_gram|tay_corr" --csv --log-file gpurun_out/r02_loc2_ncu_$loc.csv python tools/run_step.py c5 600000 --steps 1 > /dev/null 2>&1; echo ncu $loc rc=$?
done
