#!/bin/bash
set -u
O=gpurun_out
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-profile"
$B --config c0 > $O/plain_c0.log 2>&1 || exit 1
cp profiles/ncu_roofline_r02.json $O/ncu_roofline.json
for spec in "fwd_band 5 fwd_band_kernel 1" "adj_gather 5 adj_gather_kernel 1" "fgp2d 3 fgp2d_kernel 5"; do
  set -- $spec
  timeout 900 ncu --set full --import-source on --clock-control none -f -k regex:$1 -s $2 -c 1 \
      -o /tmp/ncu_c0_$3 $B --config c0 > $O/ncu_c0_$3.log 2>&1
  ncu -i /tmp/ncu_c0_$3.ncu-rep --page raw --csv > $O/raw_c0_$3.csv 2>/dev/null
  python tools/ncu_roofline.py $O/ncu_roofline.json c0 $3 $O/raw_c0_$3.csv $4
done
