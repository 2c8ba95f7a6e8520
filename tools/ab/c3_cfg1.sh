#!/bin/bash
O=gpurun_out; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_projector.py tests/test_gpu_parity_large.py tests/test_gpu_solver.py -q -x -k "3d or config3 or slice or zslab or every_forward" > $O/t_c3cfg.log 2>&1
echo "rc=$?" >> $O/t_c3cfg.log
for i in 1 2; do
  PT_FWD_CFG=100 timeout 600 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline > $O/ab_c3_old_$i.json 2>&1
  timeout 600 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline > $O/ab_c3_new_$i.json 2>&1
done
