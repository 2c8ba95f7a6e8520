#!/bin/bash
# A/B kernel timing of the in-tree build vs tools/ab/base.so on one box
O=gpurun_out; mkdir -p $O
for i in 1 2; do
  PT_LIB_OVERRIDE=$PWD/tools/ab/base.so timeout 600 python tools/kbench.py "$@" > $O/ab_base_$i.txt 2>&1
  timeout 600 python tools/kbench.py "$@" > $O/ab_new_$i.txt 2>&1
done
