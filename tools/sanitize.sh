#!/bin/bash
# compute-sanitizer sweep over every kernel of libfar.so (SURVEY.md §5 "Race detection / sanitizers").
# Usage (on the GPU box): bash tools/sanitize.sh [outdir]   -> one log per tool + summary.txt
out=${1:-gpurun_out/sanitize}
mkdir -p "$out"
: > "$out/summary.txt"
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ "$tool" = "racecheck" ] && extra="--racecheck-report all"
  args=""
  [ "$tool" != "memcheck" ] && args="--quick"   # the shared-memory trackers are ~100x slower
  timeout 2400 compute-sanitizer --tool $tool $extra --print-limit 50 --error-exitcode 9 \
    python tools/sanitize_workload.py $args > "$out/$tool.log" 2>&1
  rc=$?
  errs=$(grep -E "ERROR SUMMARY|RACECHECK SUMMARY" "$out/$tool.log" | tail -1)
  echo "$tool rc=$rc $errs $(grep -c 'sanitize workload OK' "$out/$tool.log") workload-ok" >> "$out/summary.txt"
done
cat "$out/summary.txt"
