#!/bin/bash
O=gpurun_out; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_fgp.py -q -x > $O/t_fgp.log 2>&1
echo "rc=$?" >> $O/t_fgp.log
python tools/kbench.py fgp > /dev/null 2>&1
for t in 25 17 13 30 10; do echo "tiny T=$t $(PT_FGP_T_TINY=$t timeout 300 python tools/kbench.py fgp 2>&1 | grep c0 | tr '\n' ' ')" >> $O/fgp_tiny.txt; done
echo "old 32x32 $(PT_FGP_TINY_MAX=0 timeout 300 python tools/kbench.py fgp 2>&1 | grep c0 | tr '\n' ' ')" >> $O/fgp_tiny.txt
for i in 1 2; do
  PT_FGP_TINY_MAX=0 timeout 600 python bench.py --config c0 --steps 20 --warmup 5 --no-cpu-baseline > $O/ab_c0_old_$i.json 2>&1
  timeout 600 python bench.py --config c0 --steps 20 --warmup 5 --no-cpu-baseline > $O/ab_c0_new_$i.json 2>&1
done
