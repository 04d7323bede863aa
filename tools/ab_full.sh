#!/bin/bash
# A/B of libfar builds with the secondary configs: tools/ab_full.sh a.so b.so ...
for L in "$@"; do
  FAR_LIB_OVERRIDE=$PWD/$L timeout 600 python bench.py --no-baseline --no-e2e --steps 5 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); s=d['secondary']
print('$L', round(d['value']/1e6,3), {k: round(v,3) for k,v in d['roofline']['stages_ms_per_step'].items()}, 'M3', round(s['M3_ms'],4), 'M4 A30/A100', round(s['M4_A30_streams_1024x64x64_ms'],3), round(s['M4_A100_streams_1024x64x64_ms'],3), 'BI', round(s['M5_best_improvement_100k_ms'],3), 'x4', round(s['A100x4_n64_100k_ms'],3))"
done
