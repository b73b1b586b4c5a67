#!/bin/bash
# Round profile bundle (on the GPU box): bench line, launch lists, GEMM DRAM traffic, full ncu of the top kernels.
set -x
O=gpurun_out/prof
mkdir -p $O
timeout 300 python bench.py --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/bench_launches.csv \
  python bench.py --steps 2 --warmup 3 > $O/bench_under_ncu.log 2>&1
timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --cache-control none \
  --csv --log-file $O/step.csv python tools/step_profile.py alexnet > /dev/null 2>&1
timeout 600 ncu --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
  -k regex:gemm --csv --log-file $O/gemm_traffic.csv python tools/step_profile.py alexnet > /dev/null 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:gemm_tc -c 1 -s 1 -o $O/ncu_gemm_t_wgrad \
  python tools/ncu_target.py wgrad 128 > /dev/null 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:gemm_tc -c 1 -s 1 -o $O/ncu_gemm4096 \
  python tools/ncu_target.py gemm 4096 > /dev/null 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:pack_tile -c 1 -s 1 -o $O/ncu_pack_conv1 \
  python tools/ncu_target.py pack_conv1 128 > /dev/null 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:sign_kernel -c 1 -s 1 -o $O/ncu_sign \
  python tools/ncu_target.py sign 16777216 > /dev/null 2>&1
ls -la $O
