#!/bin/bash
# corr-kernel time and roofline fraction of in-tree libraries: tools/xp_bench.sh "LIB..." CONFIG...
LIBS=$1; shift
for c in "$@"; do
  for L in $LIBS; do
    [ -f $L ] || continue
    CDMS_LIB=$L timeout 300 python bench.py --config $c --no-cpu-baseline --steps 5 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$c', '$(basename $L)', r['kernel_ms'], r['frac'])"
  done
done
