#!/bin/bash
O=gpurun_out; mkdir -p $O
python tools/kbench.py fgp3 > /dev/null 2>&1
for z in 0 32 43 52 64 86 128 0; do echo "zchunk=$z $(PT_FGP3_ZCHUNK=$z timeout 300 python tools/kbench.py fgp3 2>&1 | tr '\n' ' ')" >> $O/fgp3_zc.txt; done
