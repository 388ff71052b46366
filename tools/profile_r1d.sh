#!/bin/bash
# ncu evidence, round 1 fourth pass (run on the GPU box via gpurun; 1 GPU)
mkdir -p gpurun_out
N="ncu --set full --clock-control none --import-source on"
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/launches_r1d.csv python bench.py --steps 5 --warmup 3 --kernels none > gpurun_out/launches_bench.json 2>&1
timeout 300 $N -k regex:row_stream -s 6 -c 2 -o gpurun_out/rows_r1d python bench.py --steps 3 --warmup 3 --kernels none > /dev/null 2>&1
timeout 300 $N -k regex:attn_fwd -c 1 -o gpurun_out/attn_r1d python bench.py --steps 3 --warmup 3 --kernels sdpa > /dev/null 2>&1
timeout 300 $N -k regex:attn_fwd -c 1 -o gpurun_out/attn_rope_r1d python bench.py --steps 3 --warmup 3 --kernels sdpa_rope > /dev/null 2>&1
timeout 300 $N -k regex:"cudnn|fmha|flash" -c 1 -s 1 -o gpurun_out/torch_sdpa_r1d python tools/torch_sdpa_probe.py > /dev/null 2>&1
ls -la gpurun_out | grep r1d
