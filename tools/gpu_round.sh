#!/bin/bash
# One gpurun call: the GPU test suite and the default bench line.
#   gpurun -- bash tools/gpu_round.sh [pytest-args...]
set -u
O=gpurun_out
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -rf --durations=20 "$@" > $O/gpu_tests.log 2>&1
echo "pytest rc=$?" >> $O/gpu_tests.log
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench_c2.json 2> $O/bench_c2.err
echo "bench rc=$?" >> $O/bench_c2.err
