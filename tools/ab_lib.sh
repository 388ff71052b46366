#!/bin/bash
# A/B: time a kernel family with the regular library and with an experimental
# build (paper_2507_11978_b200/_lib/libntb200_exp.so); burst bench numbers.
K=${1:-sdpa}
python bench.py --steps 5 --warmup 3 --kernels $K 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('base', {k:(v['ms'],v['roofline']['frac']) for k,v in d['kernels'].items()})"
cp paper_2507_11978_b200/_lib/libntb200.so /tmp/base.so
cp paper_2507_11978_b200/_lib/libntb200_exp.so paper_2507_11978_b200/_lib/libntb200.so
python bench.py --steps 5 --warmup 3 --kernels $K 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('exp ', {k:(v['ms'],v['roofline']['frac']) for k,v in d['kernels'].items()})"
cp /tmp/base.so paper_2507_11978_b200/_lib/libntb200.so
