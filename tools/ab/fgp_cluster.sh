#!/bin/bash
# small-image 2D FGP in one cluster launch: region shapes (PT_FGP_CLUSTER 1-5) vs 0 (multi-launch)
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_fgp.py -q -x -k "bitwise or oracle" > $O/t_fgp_cluster.log 2>&1
echo "rc=$?" >> $O/t_fgp_cluster.log
for i in 1 2; do for m in 0 1 2 3 4 5; do
  echo "mode $m $(PT_FGP_CLUSTER=$m timeout 300 python tools/kbench.py fgp 2>&1 | grep c0 | tr '\n' ' ')" >> $O/fgp_cluster.txt
done; done
B="python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-profile"
val() { tail -1 $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'])" 2>/dev/null; }
for i in 1 2; do for m in 0 2 3 5; do
  PT_FGP_CLUSTER=$m timeout 600 $B --config c0 > /tmp/o.json 2>&1
  echo "c0 mode $m $(val /tmp/o.json)" >> $O/fgp_cluster.txt
done; done
