#!/bin/bash
# A/B of an environment knob: tools/ab_env.sh VAR=value [rounds]  (bench runs alternate: with / without)
KV="$1"; R="${2:-2}"
for r in $(seq 1 "$R"); do
  for mode in base knob; do
    if [ $mode = knob ]; then E="env $KV"; else E="env"; fi
    $E timeout 300 python bench.py --no-baseline --no-e2e --no-secondary --steps 10 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$mode', round(d['value']/1e6,3), round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['roofline']['stages_ms_per_step'].items()})"
  done
done
