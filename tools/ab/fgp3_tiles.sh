#!/bin/bash
O=gpurun_out; mkdir -p $O
python tools/kbench.py fgp3 > /dev/null 2>&1
for t in 1 2 3 4 5 0 1; do echo "triple=$t $(PT_FGP3_TRIPLE=$t timeout 300 python tools/kbench.py fgp3 2>&1 | tr '\n' ' ')" >> $O/fgp3_tiles.txt; done
timeout 600 ncu --set full --import-source on --clock-control none -f -k regex:fgp3d_col3 -s 4 -c 1 -o /tmp/p_col3 python tools/fgp3_timing.py > $O/ncu_col3.log 2>&1
ncu -i /tmp/p_col3.ncu-rep --page raw --csv > $O/raw_col3.csv 2>/dev/null
