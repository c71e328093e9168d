#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over scripts/sanitize_cases.py
# (one process per case and tool; small sizes). Logs: profiles/<tag>_sanitize_*.txt
set -u
TAG=${1:-r2}
OUT=${2:-gpurun_out}
mkdir -p "$OUT"
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in ${TOOLS:-memcheck racecheck synccheck}; do
  log="$OUT/${TAG}_sanitize_${tool}.txt"
  : > "$log"
  for c in ${CASES:-ws dense cluster kinit_mem vshard batch aux}; do
    echo "=== $tool / $c" >> "$log"
    timeout 900 $CS --tool $tool --print-limit 20 --error-exitcode 9 \
      python scripts/sanitize_cases.py $c >> "$log" 2>&1
    echo "=== $tool / $c rc=$?" >> "$log"
  done
done
