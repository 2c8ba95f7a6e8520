#!/bin/bash
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_fgp.py -q -x > $O/t_fgp3.log 2>&1
echo "rc=$?" >> $O/t_fgp3.log
for i in 1 2; do
  echo "triple $(timeout 300 python tools/kbench.py fgp3 2>&1 | tr '\n' ' ')" >> $O/fgp3_t.txt
  echo "pair   $(PT_FGP3_TRIPLE=0 timeout 300 python tools/kbench.py fgp3 2>&1 | tr '\n' ' ')" >> $O/fgp3_t.txt
done
