python -c "import __graft_entry__ as g; g.build()" || exit 1
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/r02_e1_bench_c5.json 2> gpurun_out/r02_e1_bench_c5.err; echo bench rc=$?
tail -c 3000 gpurun_out/r02_e1_bench_c5.json
timeout 600 compute-sanitizer --tool memcheck --leak-check full python tools/run_step.py c1 > gpurun_out/r02_e1_memcheck_c1.txt 2>&1; echo memcheck rc=$?
timeout 600 compute-sanitizer --tool racecheck python tools/run_step.py c1 > gpurun_out/r02_e1_racecheck_c1.txt 2>&1; echo racecheck rc=$?
timeout 600 compute-sanitizer --tool synccheck python tools/run_step.py c1 > gpurun_out/r02_e1_synccheck_c1.txt 2>&1; echo synccheck rc=$?
timeout 900 compute-sanitizer --tool memcheck python tools/run_step.py c2 20000 > gpurun_out/r02_e1_memcheck_c2.txt 2>&1; echo memcheck2 rc=$?
tail -3 gpurun_out/r02_e1_*check*.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_e1_launches_c5.csv python tools/run_step.py c5 2000000 --steps 2 > /dev/null 2>&1; echo ncu rc=$?
