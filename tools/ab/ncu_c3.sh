#!/bin/bash
set -u
O=gpurun_out
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-profile"
$B --config c3 > $O/plain_c3.log 2>&1 || exit 1
timeout 900 ncu --set full --import-source on --clock-control none -f -k regex:fgp3d_col -s 3 -c 1 \
    -o /tmp/ncu_c3_col $B --config c3 > $O/ncu_c3_col.log 2>&1
ncu -i /tmp/ncu_c3_col.ncu-rep --page raw --csv > $O/raw_c3_fgp3d_col_kernel.csv 2>/dev/null
cp profiles/ncu_roofline_r02.json $O/ncu_roofline.json
python tools/ncu_roofline.py $O/ncu_roofline.json c3 fgp3d_col_kernel $O/raw_c3_fgp3d_col_kernel.csv 50
