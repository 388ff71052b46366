#!/bin/bash
# ncu evidence, round 1 second pass (run on the GPU box via gpurun; 1 GPU)
mkdir -p gpurun_out
N="ncu --set full --clock-control none --import-source on"
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/launches_r1b.csv python bench.py --steps 5 --warmup 3 --kernels none > gpurun_out/launches_bench.json 2>&1
timeout 300 $N -k regex:row_stream -s 6 -c 2 -o gpurun_out/rows_r1b python bench.py --steps 3 --warmup 3 --kernels none > /dev/null 2>&1
timeout 300 $N -k regex:gemm_pair -c 1 -o gpurun_out/gemm_r1b python tools/one_case.py mm 4096 4096 4096 > /dev/null 2>&1
timeout 300 $N -k regex:gemm_pair -s 2 -c 1 -o gpurun_out/bmm_r1b python tools/one_case.py bmm 64 1024 1024 1024 > /dev/null 2>&1
timeout 300 $N -k regex:conv_fused -c 1 -o gpurun_out/conv_r1b python tools/one_case.py conv 64 256 56 56 256 3 3 > /dev/null 2>&1
timeout 300 $N -k regex:attn_fwd -c 1 -o gpurun_out/attn_r1b python tools/one_case.py sdpa 8 16 4096 128 > /dev/null 2>&1
timeout 300 $N -k regex:"ew_vec|rope_vec" -c 2 -o gpurun_out/ew_r1b python bench.py --steps 3 --warmup 3 --kernels add_2^24,rope > /dev/null 2>&1
ls -la gpurun_out
