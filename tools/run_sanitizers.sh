#!/bin/bash
# compute-sanitizer over every kernel instantiation (tools/sanitize_cases.py), one tool at a time.
# Logs: gpurun_out/sanitize_<tool>.log; run on a GPU box from the repo root.
set -u
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
    extra=""
    [ "$tool" = racecheck ] && extra="--racecheck-report all"
    [ "$tool" = memcheck ] && extra="--leak-check full"
    start=$(date +%s)
    timeout ${SAN_TIMEOUT:-1500} compute-sanitizer --tool $tool $extra --print-limit 200 \
        python tools/sanitize_cases.py > gpurun_out/sanitize_$tool.log 2>&1
    echo "tool=$tool rc=$? seconds=$(( $(date +%s) - start ))" >> gpurun_out/sanitize_summary.txt
    tail -3 gpurun_out/sanitize_$tool.log >> gpurun_out/sanitize_summary.txt
done
