#!/bin/bash
O=gpurun_out; mkdir -p $O
timeout 1800 python -m pytest tests/test_gpu_solver.py tests/test_gpu_multirank.py tests/test_gpu_fgp.py tests/test_gpu_parity_large.py -q -x -k "slab or zslab or fgp or config3" > $O/t_slab3.log 2>&1
echo "rc=$?" >> $O/t_slab3.log
