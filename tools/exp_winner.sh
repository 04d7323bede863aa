for b in 16 8 4 2 1; do FAR_DEBUG_WINNER_BPS=$b python bench.py --no-secondary --no-e2e --no-baseline --steps 5 > gpurun_out/w$b.log 2>&1; python -c "
import json
d=json.loads([l for l in open('gpurun_out/w$b.log') if l.startswith('{')][0]); print($b, d['ms_per_step'], round(d['roofline']['stages_ms_per_step']['winner'],3))"; done
