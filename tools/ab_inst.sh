#!/bin/bash
# A/B of an env knob across instance counts: tools/ab_inst.sh VAR=value "125000 250000 1000000" [rounds]
KV="$1"; INSTS="$2"; R="${3:-2}"
for r in $(seq 1 "$R"); do
  for I in $INSTS; do
    for mode in base knob; do
      if [ $mode = knob ]; then E="env $KV"; else E="env"; fi
      $E timeout 300 python bench.py --no-baseline --no-e2e --no-secondary --steps 10 --instances $I 2>/dev/null | tail -1 | \
        python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$I', '$mode', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['roofline']['stages_ms_per_step'].items()})"
    done
  done
done
