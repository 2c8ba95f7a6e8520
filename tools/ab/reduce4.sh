#!/bin/bash
# band reduction: one lane vs four lanes per ray (bench lines c0 c1 c2)
O=gpurun_out/reduce4.txt; : > $O
timeout 900 python -m pytest tests/test_gpu_solver.py -q -x -k "quad or pdl" > gpurun_out/t.log 2>&1; echo "pytest rc=$?" >> gpurun_out/t.log
timeout 900 python -m pytest tests/test_gpu_projector.py tests/test_gpu_parity_large.py -q -x >> gpurun_out/t.log 2>&1; echo "pytest rc=$?" >> gpurun_out/t.log
for c in c0 c1 c2; do for f in 0 1 0 1; do
  PT_FWD_REDUCE4=$f timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); kt=d['kernel_times']['fwd_reduce']; print('$c quad=$f', round(d['value'],2), round(d['e2e']['value'],2), 'reduce_us', round(1e3*kt['ms']/max(1,kt['calls']),2))" >> $O
done; done
