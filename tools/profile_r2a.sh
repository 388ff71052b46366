#!/bin/bash
# round-2 first pass (GPU box via gpurun; 1 GPU): launch list of the headline
# step, full captures of the row kernels, conv2d and sdpa_rope, racecheck of
# the CTA-pair kernels
mkdir -p gpurun_out
N="ncu --set full --clock-control none --import-source on"
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/r2a_launches.csv python bench.py --steps 5 --warmup 3 --kernels none > gpurun_out/r2a_launches_bench.json 2>&1
timeout 300 $N -k regex:row_stream -s 6 -c 2 -o gpurun_out/r2a_rows python bench.py --steps 3 --warmup 3 --kernels none > /dev/null 2>&1
timeout 300 $N -k regex:conv_fused -c 1 -o gpurun_out/r2a_conv python bench.py --steps 3 --warmup 3 --kernels conv2d > /dev/null 2>&1
timeout 300 $N -k regex:attn_fwd -c 1 -o gpurun_out/r2a_attn_rope python bench.py --steps 3 --warmup 3 --kernels sdpa_rope > /dev/null 2>&1
timeout 300 $N -k regex:"rope|ew_vec" -c 2 -o gpurun_out/r2a_ew python bench.py --steps 3 --warmup 3 --kernels silu_2^24,sdpa_rope > /dev/null 2>&1
CS="compute-sanitizer --print-limit 5 --error-exitcode 9"
for c in "mm 256 512 256" "bmm 2 256 256 128" "conv 1 64 12 12 128 3 3"; do
  echo "== racecheck: $c"; timeout 600 $CS --tool racecheck python tools/one_case.py $c 2>&1 | tail -12
done > gpurun_out/r2a_racecheck.txt
ls -la gpurun_out | grep r2a
