#!/bin/bash
# round evidence: smoke, GPU tests, bench lines (c2 + reference arm, c3, c1, c0, one-rank NCCL),
# c2 launch list, ncu roofline captures per (config, kernel)
set -u
O=gpurun_out; mkdir -p $O
bash tools/round_bench.sh
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
    --log-file $O/launches_c2.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e \
    > $O/ncu_launch.log 2>&1
bash tools/ncu_capture.sh
