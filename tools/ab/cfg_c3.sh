#!/bin/bash
O=gpurun_out; mkdir -p $O
python tools/kbench.py fwd3 > /dev/null 2>&1
for c in 100 3 0 1 2 4 5 6 7 101 100; do echo "cfg=$c $(PT_FWD_CFG=$c timeout 300 python tools/kbench.py fwd3 2>&1 | tr '\n' ' ')" >> $O/cfg_c3.txt; done
