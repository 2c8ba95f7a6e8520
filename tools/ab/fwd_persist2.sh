#!/bin/bash
O=gpurun_out; mkdir -p $O
PT_FWD_PERSIST=2 timeout 900 python -m pytest tests/test_gpu_projector.py -q -x > $O/t_fwd2.log 2>&1
echo "rc=$?" >> $O/t_fwd2.log
python tools/kbench.py fwd > /dev/null 2>&1
for v in 0 1 2; do for ips in 2 4 10; do echo "persist=$v ips=$ips $(PT_FWD_PERSIST=$v PT_FWD_IPS=$ips timeout 600 python tools/kbench.py fwd 2>&1 | tr '\n' ' ')" >> $O/ab_p.txt; done; done
