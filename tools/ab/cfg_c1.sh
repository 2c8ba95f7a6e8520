#!/bin/bash
O=gpurun_out; mkdir -p $O
python tools/kbench.py fwd > /dev/null 2>&1
for c in 3 0 1 2 4 5 6 7 100 101 3; do echo "cfg=$c $(PT_FWD_CFG=$c timeout 300 python tools/kbench.py fwd 2>&1 | tr '\n' ' ')" >> $O/cfg_c1.txt; done
