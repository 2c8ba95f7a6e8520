#!/bin/bash
O=gpurun_out; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_fgp.py tests/test_gpu_rows.py -q -x > $O/t_fgpcl.log 2>&1
echo "rc=$?" >> $O/t_fgpcl.log
python tools/kbench.py fgp > /dev/null 2>&1
for v in 2 1 2 1; do echo "cluster=$v $(PT_FGP_CLUSTER=$v timeout 300 python tools/kbench.py fgp 2>&1 | tr '\n' ' ')" >> $O/fgp_cl.txt; done
for t in 6 10 12; do echo "cluster=2 T=$t $(PT_FGP_T=$t timeout 300 python tools/kbench.py fgp 2>&1 | tr '\n' ' ')" >> $O/fgp_cl.txt; done
