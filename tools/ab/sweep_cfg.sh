#!/bin/bash
# gather tiles (c1, c3) and forward waves (c1, c0) on bench lines
O=gpurun_out; mkdir -p $O
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-profile"
val() { tail -1 $1 | python -c "import json,sys; print(json.loads(sys.stdin.read())['value'])" 2>/dev/null; }
for c in c1 c3; do for t in d 0 1 2 3; do
  if [ $t = d ]; then timeout 600 $B --config $c > /tmp/o.json 2>&1; else PT_GATHER_TILE=$t timeout 600 $B --config $c > /tmp/o.json 2>&1; fi
  echo "$c gather_tile=$t $(val /tmp/o.json)" >> $O/sweep_cfg.txt
done; done
for c in c1 c0; do for w in d 2 4 6; do
  if [ $w = d ]; then timeout 600 $B --config $c > /tmp/o.json 2>&1; else PT_FWD_WAVES=$w timeout 600 $B --config $c > /tmp/o.json 2>&1; fi
  echo "$c fwd_waves=$w $(val /tmp/o.json)" >> $O/sweep_cfg.txt
done; done
