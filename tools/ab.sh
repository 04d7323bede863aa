#!/bin/bash
# A/B timing of two libfar builds on the GPU box: tools/ab.sh a.so b.so [rounds]
A=$1; B=$2; R=${3:-3}
for r in $(seq 1 $R); do
  for L in $A $B; do
    FAR_LIB_OVERRIDE=$PWD/$L timeout 300 python bench.py --no-baseline --no-e2e --no-secondary --steps 5 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$L', round(d['value']/1e6,3), round(d['ms_per_step'],3))"
  done
done
