python -c "import __graft_entry__ as g; g.build()" || exit 1
mkdir -p gpurun_out
timeout 900 ncu --set full --cache-control none --clock-control none -k regex:"tay_corr" -s 2 -c 1 -o gpurun_out/r02_w5 python tools/run_step.py c5 600000 --steps 3 > gpurun_out/r02_w5.log 2>&1; echo ncu rc=$?
