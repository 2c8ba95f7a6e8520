#!/bin/bash
# 2D FGP on small images: strip height x T (kbench fgp: c0 FGP-50 at 128^2)
O=gpurun_out/fgp_small.txt; : > $O
python tools/kbench.py fgp > /dev/null 2>&1
for sh in 8 4 2; do for t in 6 8 10 12; do
  echo "strip=$sh T=$t $(PT_FGP_SMALL_STRIP=$sh PT_FGP_T_SMALL=$t python tools/kbench.py fgp 2>/dev/null | grep c0 | tr '\n' ' ')" >> $O
done; done
