#!/bin/bash
# winner-stage A/B: libs x blocks per SM (FAR_DEBUG_WINNER_BPS) at 1M and 125k M5 instances
for r in 1 2; do
for L in abl/base.so abl/pool.so; do for B in 16 8 24; do for I in 1000000 125000; do
  FAR_DEBUG_WINNER_BPS=$B FAR_LIB_OVERRIDE=$PWD/$L timeout 300 python bench.py --no-baseline --no-e2e --no-secondary --steps 10 --instances $I 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); s=d['roofline']['stages_ms_per_step']; print('$L', 'bps=$B', $I, round(d['ms_per_step'],3), 'winner', round(s['winner'],3))"
done; done; done; done
