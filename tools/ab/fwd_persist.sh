#!/bin/bash
# persistent producer/consumer forward vs tools/ab/base.so: projector tests + forward timings
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_projector.py tests/test_gpu_parity_large.py -q -x -k "not config3 and not two_epochs" > $O/t_fwd.log 2>&1
echo "rc=$?" >> $O/t_fwd.log
for i in 1 2; do
  PT_LIB_OVERRIDE=$PWD/tools/ab/base.so timeout 600 python tools/kbench.py fwd fwd3 > $O/ab_base_$i.txt 2>&1
  timeout 600 python tools/kbench.py fwd fwd3 > $O/ab_new_$i.txt 2>&1
done
for ips in 4 6 16 24; do echo "ips=$ips $(PT_FWD_IPS=$ips timeout 600 python tools/kbench.py fwd fwd3 2>&1 | tr '\n' ' ')" >> $O/ab_ips.txt; done
