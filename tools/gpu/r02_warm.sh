python -c "import __graft_entry__ as g; g.build()" || exit 1
mkdir -p gpurun_out
for loc in 0 1; do
CDMS_LOCALITY=$loc timeout 900 ncu --set full --cache-control none --clock-control none -k regex:"tay_gram|tay_corr" -s 4 -c 2 -o gpurun_out/r02_warm_$loc python tools/run_step.py c5 600000 --steps 3 > gpurun_out/r02_warm_$loc.log 2>&1; echo ncu $loc rc=$?
done
