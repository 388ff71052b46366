#!/bin/bash
# Alternate bench runs of a kernel family over in-tree library variants
# (libntb200_<tag>.so, selected by NTB_LIB_VARIANT; "base" = libntb200.so).
# usage: tools/var_sweep.sh KERNELS ROUNDS TAG...   (library reference ops skipped)
K=$1; R=$2; shift 2
export NTB_BENCH_TORCH=0
for r in $(seq $R); do
  for v in "$@"; do
    if [ "$v" = base ]; then unset NTB_LIB_VARIANT; else export NTB_LIB_VARIANT=$v; fi
    python bench.py --steps 5 --warmup 3 --kernels $K 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('$v', {k:(round(v['ms'],4),v['roofline']['frac'],v['verify']['ok']) for k,v in d['kernels'].items()})"
  done
done
