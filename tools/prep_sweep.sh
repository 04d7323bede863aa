#!/bin/bash
# prep occupancy sweep (blocks of 4 warps per SM; the launch bounds allow 8)
for r in 1 2; do for B in 8 7 6; do
  FAR_DEBUG_PREP_BPS=$B timeout 300 python bench.py --no-baseline --no-e2e --no-secondary --steps 10 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bps=$B', round(d['ms_per_step'],3), 'prep', round(d['roofline']['stages_ms_per_step']['prep'],3))"
done; done
