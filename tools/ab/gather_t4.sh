#!/bin/bash
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_projector.py -q -x -k "gather_tile" > $O/t_g4.log 2>&1
echo "rc=$?" >> $O/t_g4.log
B="python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-profile --config c0"
val() { tail -1 $1 | python -c "import json,sys; print(json.loads(sys.stdin.read())['value'])" 2>/dev/null; }
for i in 1 2; do for t in d 4 3; do
  if [ $t = d ]; then timeout 600 $B > /tmp/o.json 2>&1; else PT_GATHER_TILE=$t timeout 600 $B > /tmp/o.json 2>&1; fi
  echo "c0 gather_tile=$t $(val /tmp/o.json)" >> $O/g4.txt
done; done
