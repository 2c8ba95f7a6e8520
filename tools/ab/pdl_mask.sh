#!/bin/bash
# PDL release point per kernel family (tools/ab/build_pdl_variants.sh builds the
# variants): base.so = release at kernel end, no pre-wait loads in fwd_reduce;
# in-tree = release at kernel end + fwd_reduce's static loads before its wait;
# pdl_<mask>.so = families in <mask> release right after their own wait
# (1 fwd_band, 2 fwd_small, 4 fwd_reduce, 8 gather, 16 fgp2d, 32 fgp3d, 64 others).
O=gpurun_out; mkdir -p $O
B="python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-profile --no-e2e"
val() { tail -1 $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'])" 2>/dev/null; }
run() { # label lib configs...
  local label=$1 lib=$2; shift 2
  for c in "$@"; do
    PT_LIB_OVERRIDE=$lib timeout 600 $B --config $c > /tmp/o.json 2>&1
    echo "$c $label $(val /tmp/o.json)" >> $O/pdl_mask.txt
  done
}
for i in 1 2; do
  run base $PWD/tools/ab/base.so c2 c1 c0 c3
  run tree "" c2 c1 c0 c3
  for m in 1 2 3 4 16 19 127; do run m$m $PWD/tools/ab/pdl_$m.so c2 c1 c0; done
  run m32 $PWD/tools/ab/pdl_32.so c3
done
sort -s -k1,1 $O/pdl_mask.txt
