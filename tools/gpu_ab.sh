# A/B bench of the current tree (new prep) vs FAR_OLD_PREP=1, then the GPU suite (round-2 dev helper)
python bench.py --no-secondary --no-e2e --no-baseline > gpurun_out/bench_new.log 2>&1
FAR_OLD_PREP=1 python bench.py --no-secondary --no-e2e --no-baseline > gpurun_out/bench_old.log 2>&1
for f in bench_new bench_old; do python - "$f" <<'PY'
import json,sys
l=[x for x in open(f"gpurun_out/{sys.argv[1]}.log") if x.startswith("{")]
if l:
    d=json.loads(l[0]); print(sys.argv[1], d["value"], d["ms_per_step"], d["roofline"]["stages_ms_per_step"])
else: print(open(f"gpurun_out/{sys.argv[1]}.log").read()[-2000:])
PY
done
if [ -n "$NCU" ]; then ncu --set full --clock-control none --import-source on -k regex:$NCU -s 1 -c 1 -o gpurun_out/$NCU python bench.py --instances 200000 --steps 1 --warmup 1 --profile-run --no-secondary > gpurun_out/ncu_$NCU.log 2>&1; fi
if [ -z "$NOTEST" ]; then timeout 900 python -m pytest tests -m gpu -x -q $TESTS > gpurun_out/gputest.log 2>&1; tail -3 gpurun_out/gputest.log; fi
