#!/usr/bin/env bash
# compute-sanitizer over every kernel family of libgpoeo.so (tools/sanitize_workload.py).
# Usage (on a GPU box): bash tools/sanitize.sh [outdir]   -> <outdir>/sanitize_<tool>_<case>.log
# and <outdir>/sanitize_summary.txt (one line per run: tool, case, exit code, error summary).
set -u
OUT=${1:-gpurun_out}
mkdir -p "$OUT"
SUM="$OUT/sanitize_summary.txt"
: > "$SUM"
CS=${COMPUTE_SANITIZER:-compute-sanitizer}
for tool in memcheck racecheck synccheck initcheck; do
  for case in cfg1 cfg2 scorer fused cluster band; do
    log="$OUT/sanitize_${tool}_${case}.log"
    extra=""
    [ "$tool" = racecheck ] && extra="--racecheck-report all"
    timeout 900 "$CS" --tool "$tool" $extra --error-exitcode 99 --target-processes all \
      python tools/sanitize_workload.py "$case" > "$log" 2>&1
    rc=$?
    summary=$(grep -E "ERROR SUMMARY|RACECHECK SUMMARY|LEAK SUMMARY" "$log" | tr '\n' ' ')
    echo "$tool $case rc=$rc $summary" | tee -a "$SUM"
  done
done
