#!/bin/bash
# M3 secondary A/B: tools/ab_m3.sh a.so b.so ... (M3 100k x n=32 ms from the bench's secondary block)
for L in "$@"; do
  FAR_LIB_OVERRIDE=$PWD/$L timeout 300 python bench.py --no-baseline --no-e2e --steps 3 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$L M3_ms', round(d['secondary']['M3_ms'],4))"
done
