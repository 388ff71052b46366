#!/bin/bash
# round-2 closing evidence pass (GPU box via gpurun; 1 GPU): after the register splits, PDL attention,
# (attention 72/216, 3xTF32 72/216) - the bench line, the reference arm, the GPU tests +
# smoke, the headline launch list, per-kernel traffic, and full captures of
# the attention kernel at the BASELINE and the paper shapes
mkdir -p gpurun_out
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_write.sum"
N="ncu --set full --clock-control none --import-source on"
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/r2f_gputest.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2f_smoke.txt 2>&1
timeout 600 python bench.py > gpurun_out/r2f_bench.json 2> gpurun_out/r2f_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2f_ref.json 2> gpurun_out/r2f_ref.err
timeout 300 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/r2f_launches.csv \
  python bench.py --steps 5 --warmup 3 --kernels none > gpurun_out/r2f_launches_bench.json 2>&1
timeout 600 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/r2f_traffic.csv \
  python tools/traffic_probe.py > gpurun_out/r2f_traffic_order.txt 2>&1
timeout 600 $N -k regex:attn_fwd -c 1 -o gpurun_out/r2f_attn python tools/attn_once.py 32 32 4096 128 > /dev/null 2>&1
timeout 300 $N -k regex:attn_fwd -c 1 -o gpurun_out/r2f_attn_paper python tools/attn_once.py 4 48 1024 64 > /dev/null 2>&1
timeout 300 $N -k regex:gemm_tf32 -c 1 -o gpurun_out/r2f_tf32 python tools/tf32_time.py > /dev/null 2>&1
ls -la gpurun_out | grep "r2f_"
