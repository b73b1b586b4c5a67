#!/bin/bash
# Round-2 profile bundle (on the GPU box): bench line, launch list, per-launch DRAM traffic of the step's
# GEMM / sign launches, per-launch breakdowns of the three workloads.  Outputs under gpurun_out/prof.
set -x
O=gpurun_out/prof
mkdir -p $O
timeout 400 python bench.py > $O/bench.json 2> $O/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file $O/bench_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-side --no-cpu-baseline --no-e2e > $O/bench_under_ncu.log 2>&1
timeout 600 ncu --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
  -k regex:gemm --csv --log-file $O/gemm_traffic.csv python tools/step_profile.py alexnet > /dev/null 2>&1
timeout 600 ncu --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
  -k regex:sign --csv --log-file $O/sign_traffic.csv python tools/step_profile.py alexnet > /dev/null 2>&1
timeout 300 python tools/step_breakdown.py alexnet > $O/breakdown_alexnet.txt 2>&1
timeout 600 python tools/step_breakdown.py resnet50 64 > $O/breakdown_resnet50_b64.txt 2>&1
timeout 300 python tools/step_breakdown.py resnet50 1 > $O/breakdown_resnet50_b1.txt 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:sign_kernel -c 1 -s 1 -o $O/ncu_sign \
  python tools/ncu_target.py sign 16777216 > /dev/null 2>&1
ls -la $O
