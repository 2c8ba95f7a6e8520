#!/bin/bash
# 2D FGP region shapes x iterations per launch (kbench fgp), one box
O=gpurun_out/fgp_shape.txt; : > $O
python tools/kbench.py fgp > /dev/null 2>&1  # warm the box
for sh in 0 1 2; do for t in 6 8 10 12; do
  echo "shape=$sh T=$t $(PT_FGP_SHAPE=$sh PT_FGP_T=$t python tools/kbench.py fgp 2>/dev/null | tr '\n' ' ')" >> $O
done; done
