#!/bin/bash
# small-image fused forward vs tools/ab/base.so: tests + c0 bench
O=gpurun_out; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x > $O/t_small.log 2>&1
echo "rc=$?" >> $O/t_small.log
for i in 1 2; do
  PT_LIB_OVERRIDE=$PWD/tools/ab/base.so timeout 600 python bench.py --config c0 --steps 20 --warmup 5 --no-cpu-baseline > $O/ab_c0_base_$i.json 2>&1
  timeout 600 python bench.py --config c0 --steps 20 --warmup 5 --no-cpu-baseline > $O/ab_c0_new_$i.json 2>&1
done
