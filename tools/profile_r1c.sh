#!/bin/bash
# ncu evidence, round 1 third pass (run on the GPU box via gpurun; 1 GPU)
mkdir -p gpurun_out
N="ncu --set full --clock-control none --import-source on"
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/launches_r1c.csv python bench.py --steps 5 --warmup 3 --kernels none > gpurun_out/launches_bench.json 2>&1
timeout 300 $N -k regex:gemm_pair -c 1 -o gpurun_out/gemm_r1c python tools/one_case.py mm 4096 4096 4096 > /dev/null 2>&1
timeout 300 $N -k regex:conv_fused -c 1 -o gpurun_out/conv_r1c python tools/one_case.py conv 64 256 56 56 256 3 3 > /dev/null 2>&1
timeout 300 $N -k regex:attn_fwd -c 1 -o gpurun_out/attn_r1c python tools/one_case.py sdpa 8 16 4096 128 > /dev/null 2>&1
ls -la gpurun_out
