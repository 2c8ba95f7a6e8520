#!/bin/bash
# 2D FGP: packed edge regions (per-half selects) vs tools/ab/base.so (scalar edge path)
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_fgp.py tests/test_gpu_rows.py -q -x > $O/t_fgp_edge.log 2>&1
echo "rc=$?" >> $O/t_fgp_edge.log
for i in 1 2; do
  echo "base $(PT_LIB_OVERRIDE=$PWD/tools/ab/base.so timeout 300 python tools/kbench.py fgp 2>&1 | tr '\n' ' ')" >> $O/fgp_edge.txt
  echo "new  $(timeout 300 python tools/kbench.py fgp 2>&1 | tr '\n' ' ')" >> $O/fgp_edge.txt
done
B="python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-profile"
val() { tail -1 $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'])" 2>/dev/null; }
for i in 1 2; do for c in c2 c1 c0; do
  PT_LIB_OVERRIDE=$PWD/tools/ab/base.so timeout 600 $B --config $c > /tmp/o.json 2>&1
  echo "$c base $(val /tmp/o.json)" >> $O/fgp_edge.txt
  timeout 600 $B --config $c > /tmp/o.json 2>&1
  echo "$c new  $(val /tmp/o.json)" >> $O/fgp_edge.txt
done; done
