#!/bin/bash
# compute-sanitizer passes over one small case per kernel family (GPU box)
CS="compute-sanitizer --print-limit 5 --error-exitcode 9"
run() { echo "== $1: $2"; timeout 600 $CS --tool $1 python tools/one_case.py $2 2>&1 | grep -E "ERROR SUMMARY|max err|Error|error" | head -6; }
for tool in memcheck racecheck synccheck initcheck; do
  run $tool "ew 100003"
  run $tool "rows 64 4096"
  run $tool "rope 1 128 2 128"
  run $tool "mm 256 512 256"
  run $tool "bmm 2 256 256 128"
  run $tool "conv 1 64 12 12 128 3 3"
  run $tool "sdpa 1 2 300 128"
  run $tool "sdpa 1 2 200 64"
done
