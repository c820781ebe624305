#!/bin/bash
# compute-sanitizer over tools/sanitize_case.py, ONE tool per invocation (the
# B200 profiling guide: several tools in one call once left a GPU unusable).
#   tools/sanitize.sh memcheck|racecheck|initcheck|synccheck
# The plain run must pass first; the log goes to gpurun_out/sanitize_<tool>.log.
set -e
tool=${1:-memcheck}
mkdir -p gpurun_out
timeout 600 python tools/sanitize_case.py > gpurun_out/sanitize_plain.log 2>&1
extra=""
# (no --leak-check: torch keeps its cached allocations until exit)
[ "$tool" = "racecheck" ] && extra="--racecheck-report analysis"
timeout 2400 compute-sanitizer --tool $tool $extra --target-processes all --print-limit 50 \
    python tools/sanitize_case.py > gpurun_out/sanitize_$tool.log 2>&1 || true
tail -5 gpurun_out/sanitize_$tool.log
