#!/bin/bash
# Round-2 end-of-session profile bundle (GPU box): bench line, launch list, per-launch DRAM traffic of the
# step's GEMM / sign launches, per-launch breakdowns of the four workloads.  Outputs under gpurun_out/prof2.
set -x
O=gpurun_out/prof2
mkdir -p $O
timeout 400 python bench.py > $O/bench.json 2> $O/bench.err
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file $O/bench_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-side --no-cpu-baseline --no-e2e > $O/bench_under_ncu.log 2>&1
timeout 600 ncu --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
  -k regex:gemm --csv --log-file $O/gemm_traffic.csv python tools/step_profile.py alexnet > /dev/null 2>&1
timeout 600 ncu --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
  -k regex:sign --csv --log-file $O/sign_traffic.csv python tools/step_profile.py alexnet > /dev/null 2>&1
timeout 300 python tools/step_breakdown.py alexnet > $O/breakdown_alexnet.txt 2>&1
timeout 600 python tools/step_breakdown.py resnet50 64 > $O/breakdown_resnet50_b64.txt 2>&1
timeout 300 python tools/step_breakdown.py resnet50 1 > $O/breakdown_resnet50_b1.txt 2>&1
timeout 300 python tools/step_breakdown.py vgg16 32 > $O/breakdown_vgg16_b32.txt 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:sign2_kernel -c 1 -s 1 -o $O/ncu_sign2 \
  python tools/ncu_target.py sign 49152 > /dev/null 2>&1
ls -la $O
