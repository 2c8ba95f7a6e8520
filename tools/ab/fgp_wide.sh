#!/bin/bash
# 2D FGP region shapes: PT_FGP_WIDE 0 (64x64, 512 thr, 2 CTA/SM), 1 (128x64, 1024 thr),
# 2 (96x64, 768 thr), 3 (128x32 4-row strips, 1024 thr) x T
O=gpurun_out; mkdir -p $O
PT_FGP_WIDE=1 timeout 900 python -m pytest tests/test_gpu_fgp.py -q -x -k "bitwise or oracle" > $O/t_fgp_wide.log 2>&1
echo "rc=$?" >> $O/t_fgp_wide.log
for w in 0 1 2 3; do for t in 6 8 10 12; do
  echo "wide $w T $t $(PT_FGP_WIDE=$w PT_FGP_T=$t timeout 300 python tools/kbench.py fgp 2>&1 | grep -v c0 | tr '\n' ' ')" >> $O/fgp_wide.txt
done; done
