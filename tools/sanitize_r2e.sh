#!/bin/bash
# compute-sanitizer on the attention kernel after the late round-2 changes
# (72/216 register split, PDL launch, per-D P chunks, pv_done consumed every
# tile), plain and rope, D = 64 / 128, single- and multi-unit schedules
# (GPU box; output summarised in profiles/r2e_sanitizer.txt)
CS="compute-sanitizer --print-limit 3"
for c in "sdpa 1 2 300 128" "sdpa 1 2 200 64" "sdpa 2 40 520 64" "sdpa 2 80 300 128" "sdpa_rope 2 300 3 128" "sdpa_rope 2 600 3 64"; do
  for tool in memcheck synccheck; do
    echo "=== $tool $c"; timeout 600 $CS --tool $tool python tools/one_case.py $c 2>&1 | grep -v "Host Frame" | grep -E "max err|SUMMARY" | cut -c1-60 | head -3
  done
done
for c in "sdpa 1 2 300 128" "sdpa 2 40 520 64" "sdpa 2 80 300 128" "sdpa_rope 2 600 3 64"; do
  echo "=== racecheck $c"; timeout 600 $CS --tool racecheck python tools/one_case.py $c 2>&1 | grep -v "Host Frame" | grep -E "max err|SUMMARY|Race reported|and Write" | cut -c1-240 | head -4
done
for tool in memcheck synccheck; do
  echo "=== $tool mm32 256 512 256"; timeout 600 $CS --tool $tool python tools/one_case.py mm32 256 512 256 2>&1 | grep -E "max err|SUMMARY" | head -3
done
