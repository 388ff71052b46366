#!/bin/bash
# compute-sanitizer on the attention kernel after the late round-2 changes
# (72/216 register split, PDL launch, P chunks per D, per-chunk sdpa_rope)
# and on the 3xTF32 kernel (register split); GPU box, small cases
CS="compute-sanitizer --print-limit 5 --error-exitcode 9"
run() { echo "== $1: $2"; timeout 900 $CS --tool $1 python tools/one_case.py $2 2>&1 | grep -E "ERROR SUMMARY|max err|Error|error" | head -6; }
for tool in memcheck racecheck synccheck; do
  run $tool "sdpa 1 2 300 128"
  run $tool "sdpa 1 2 200 64"
  run $tool "sdpa 2 40 520 64"
  run $tool "sdpa_rope 2 300 3 128"
  run $tool "sdpa_rope 1 256 2 64"
done
for tool in memcheck synccheck; do
  run $tool "mm32 256 512 256"
done
