for r in 1 2; do for mode in base knob; do
 if [ $mode = knob ]; then E="env FAR_DEBUG_NO_ROUND_BALANCE=1"; else E="env"; fi
 $E timeout 300 python bench.py --no-baseline --no-e2e --steps 5 --instances 125000 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); s=d['secondary']; print('$mode', round(d['ms_per_step'],3), round(d['roofline']['stages_ms_per_step']['members'],3), 'M3', round(s['M3_ms'],4), 'M4', round(s.get('M4_A100_streams_1024x64x64_ms',0),3))"
done; done
