#!/bin/bash
# ncu captures of the dominant kernels on bench.py's own workloads (one launch
# each, after the same command ran clean without ncu), digested into
# gpurun_out/ncu_roofline.json by tools/ncu_roofline.py.  Run under gpurun.
set -u
O=gpurun_out; mkdir -p $O
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-profile"
cap() {  # config regex skip name per_call
  local cfg=$1 rx=$2 skip=$3 name=$4 pc=$5
  # reports stay on the box (/tmp): only the raw CSV digests come back (gpurun_out <= 64 MiB)
  timeout 900 ncu --set full --import-source on --clock-control none -f -k regex:$rx -s $skip -c 1 \
      -o /tmp/ncu_${cfg}_${name} $B --config $cfg > $O/ncu_${cfg}_${name}.log 2>&1
  ncu -i /tmp/ncu_${cfg}_${name}.ncu-rep --page raw --csv > $O/raw_${cfg}_${name}.csv 2>/dev/null
  python tools/ncu_roofline.py $O/ncu_roofline.json $cfg $name $O/raw_${cfg}_${name}.csv $pc
}
for cfg in c2 c3 c1 c0; do
  $B --config $cfg > $O/plain_$cfg.log 2>&1 || { echo "plain run $cfg failed"; continue; }
done
cap c2 fwd_band 5 fwd_band_kernel 1
cap c2 adj_gather 5 adj_gather_kernel 1
cap c2 fgp2d 3 fgp2d_kernel 13
cap c3 fgp3d_col3 3 fgp3d_col3_kernel 33
cap c3 fwd_band 5 fwd_band_kernel 1
cap c1 fwd_band 5 fwd_band_kernel 1
cap c1 adj_gather 5 adj_gather_kernel 1
cap c1 fgp2d 3 fgp2d_kernel 15
cap c0 fwd_small 5 fwd_small_kernel 1
cap c0 adj_gather 5 adj_gather_kernel 1
cap c0 fgp2d 3 fgp2d_kernel 7
