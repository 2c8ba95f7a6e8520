#!/bin/bash
# PDL: successors released right after each kernel's own wait (in-tree build)
# vs at the end of each kernel (tools/ab/base.so, -DPT_PDL_LATE behaviour).
O=gpurun_out; mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q -x > $O/t_pdl_early.log 2>&1
echo "rc=$?" >> $O/t_pdl_early.log
B="python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-profile"
val() { tail -1 $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'])" 2>/dev/null; }
for i in 1 2; do for c in c2 c0 c1 c3; do
  PT_LIB_OVERRIDE=$PWD/tools/ab/base.so timeout 600 $B --config $c > /tmp/o.json 2>&1
  echo "$c base $(val /tmp/o.json)" >> $O/pdl_early.txt
  timeout 600 $B --config $c > /tmp/o.json 2>&1
  echo "$c new  $(val /tmp/o.json)" >> $O/pdl_early.txt
done; done
for i in 1 2; do
  echo "base $(PT_LIB_OVERRIDE=$PWD/tools/ab/base.so timeout 300 python tools/kbench.py fgp 2>&1 | tr '\n' ' ')" >> $O/pdl_early.txt
  echo "new  $(timeout 300 python tools/kbench.py fgp 2>&1 | tr '\n' ' ')" >> $O/pdl_early.txt
done
cat $O/pdl_early.txt; tail -3 $O/t_pdl_early.log
