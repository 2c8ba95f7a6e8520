#!/bin/bash
# step gathers split over angle parts + combine/epilogue kernel (PT_STEP_SPLIT) on c1 / c0
O=gpurun_out/step_split.txt; : > $O
for c in c1 c0; do for k in 0 2 3 4 0; do
  PT_STEP_SPLIT=$k timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c split=$k', round(d['value'],1), round(d['e2e']['value'],1))" >> $O
done; done
