#!/bin/bash
# round-2 second evidence pass (GPU box via gpurun; 1 GPU): the bench line,
# the reference arm, the headline launch list, per-kernel traffic, and full
# captures of the kernels changed in this pass (streaming elementwise,
# attention at the paper shape with the single-tile tail units)
mkdir -p gpurun_out
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_write.sum"
N="ncu --set full --clock-control none --import-source on"
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/r2b_gputest.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2b_smoke.txt 2>&1
timeout 600 python bench.py > gpurun_out/r2b_bench.json 2> gpurun_out/r2b_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2b_ref.json 2> gpurun_out/r2b_ref.err
timeout 300 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/r2b_launches.csv \
  python bench.py --steps 5 --warmup 3 --kernels none > gpurun_out/r2b_launches_bench.json 2>&1
timeout 600 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/r2b_traffic.csv \
  python tools/traffic_probe.py > gpurun_out/r2b_traffic_order.txt 2>&1
timeout 300 $N -k regex:ew_stream -c 2 -o gpurun_out/r2b_ew python tools/traffic_probe.py > /dev/null 2>&1
timeout 300 $N -k regex:attn_fwd -c 1 -o gpurun_out/r2b_attn_paper python tools/attn_once.py 4 48 1024 64 > /dev/null 2>&1
ls -la gpurun_out | grep "r2b_"
