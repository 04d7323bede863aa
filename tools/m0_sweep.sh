#!/bin/bash
# member0 occupancy sweep (n > 64): warps per SM x block size, 1M M5
for r in 1 2; do for TB in 128 64; do for W in 8 10 12; do
  FAR_DEBUG_M0_TB=$TB FAR_DEBUG_M0_WARPS=$W timeout 300 python bench.py --no-baseline --no-e2e --no-secondary --steps 10 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('tb=$TB warps=$W', round(d['ms_per_step'],3), 'member0', round(d['roofline']['stages_ms_per_step']['member0'],3))"
done; done; done
