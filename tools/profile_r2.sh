#!/bin/bash
# round-2 final evidence pass (GPU box via gpurun; 1 GPU)
mkdir -p gpurun_out
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_write.sum"
N="ncu --set full --clock-control none --import-source on"
timeout 600 python bench.py > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2_ref.json 2> gpurun_out/r2_ref.err
timeout 300 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/r2_launches.csv \
  python bench.py --steps 5 --warmup 3 --kernels none > gpurun_out/r2_launches_bench.json 2>&1
timeout 600 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/r2_traffic.csv \
  python tools/traffic_probe.py > gpurun_out/r2_traffic_order.txt 2>&1
timeout 300 $N -k regex:row_stream -c 2 -o gpurun_out/r2_rows python tools/traffic_probe.py > /dev/null 2>&1
timeout 300 $N -k regex:ew_vec -c 3 -o gpurun_out/r2_ew python tools/traffic_probe.py > /dev/null 2>&1
timeout 300 $N -k regex:gemm_pair -c 1 -o gpurun_out/r2_gemm python tools/traffic_probe.py > /dev/null 2>&1
timeout 300 $N -k regex:gemm_tf32 -c 1 -o gpurun_out/r2_gemm_tf32 python tools/traffic_probe.py > /dev/null 2>&1
timeout 300 $N -k regex:conv_fused -c 1 -o gpurun_out/r2_conv python tools/traffic_probe.py > /dev/null 2>&1
timeout 300 $N -k regex:attn_fwd -c 1 -o gpurun_out/r2_attn python tools/traffic_probe.py > /dev/null 2>&1
ls -la gpurun_out | grep "r2_"
