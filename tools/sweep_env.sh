#!/bin/bash
# env sweep of one libfar build on the GPU box: tools/sweep_env.sh lib.so "ENV1=a ENV2=b" "ENV1=c" ...
L=$1; shift
for E in "$@"; do
  env $E FAR_LIB_OVERRIDE=$PWD/$L timeout 300 python bench.py --no-baseline --no-e2e --no-secondary --steps 5 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$E', round(d['value']/1e6,3), {k: round(v,3) for k,v in d['roofline']['stages_ms_per_step'].items()})"
done
