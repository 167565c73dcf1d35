#!/bin/bash
# A/B the corr kernel of two in-tree libraries on the same box: tools/ab_bench.sh LIB_A LIB_B CONFIG...
# prints config, library, step ms, corr kernel ms, roofline frac (3 alternating runs each)
A=$1; B=$2; shift 2
for c in "$@"; do
  for r in 1 2 3; do
    for L in $A $B; do
      CDMS_LIB=$L timeout 300 python bench.py --config $c --no-cpu-baseline --steps 5 2>/dev/null | tail -1 | \
        python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$c', '$(basename $L)', round(d['ms_per_step'],4), r['kernel_ms'], r['frac'])"
    done
  done
done
