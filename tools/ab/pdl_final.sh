#!/bin/bash
# The kept PDL setting (in-tree: the small forward releases early) against
# base.so (every release at kernel end) and two wider masks; then the GPU suite.
O=gpurun_out; mkdir -p $O
B="python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-profile"
val() { tail -1 $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'])" 2>/dev/null; }
run() { local label=$1 lib=$2; shift 2
  for c in "$@"; do
    PT_LIB_OVERRIDE=$lib timeout 600 $B --config $c > /tmp/o.json 2>&1
    echo "$c $label $(val /tmp/o.json)" >> $O/pdl_final.txt
  done; }
for i in 1 2; do
  run base $PWD/tools/ab/base.so c0 c1 c2 c3
  run tree "" c0 c1 c2 c3
  run m10 $PWD/tools/ab/pdl_10.so c0 c1
  run m66 $PWD/tools/ab/pdl_66.so c0 c1
done
sort -s -k1,1 $O/pdl_final.txt
timeout 2400 python -m pytest tests -m gpu -q -x > $O/t_pdl_final.log 2>&1
echo "rc=$?" >> $O/t_pdl_final.log; tail -3 $O/t_pdl_final.log
