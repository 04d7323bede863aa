#!/bin/bash
# per-stage A/B: tools/ab_stages.sh a.so b.so ... (one bench run each, stage split printed)
for L in "$@"; do
  FAR_LIB_OVERRIDE=$PWD/$L timeout 300 python bench.py --no-baseline --no-e2e --no-secondary --steps 5 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$L', round(d['value']/1e6,3), {k: round(v,3) for k,v in d['roofline']['stages_ms_per_step'].items()})"
done
