#!/bin/bash
# One GPU call's worth of round evidence (run under gpurun from the repo root):
#   bench c2 (+ cpu baseline), reference arm, c3 bench, launch list of the c2 bench,
#   ncu --set full of the top kernels (one launch each).  Outputs in gpurun_out/.
set -u
O=gpurun_out
timeout 900 python bench.py > $O/bench_c2.json 2> $O/bench_c2.err
timeout 900 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err
timeout 600 python bench.py --config c3 --no-cpu-baseline > $O/bench_c3.json 2> $O/bench_c3.err
timeout 600 python bench.py --config c1 --no-cpu-baseline > $O/bench_c1.json 2> $O/bench_c1.err
timeout 600 python bench.py --config c0 --no-cpu-baseline > $O/bench_c0.json 2> $O/bench_c0.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
    --log-file $O/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e \
    > $O/ncu_launch.log 2>&1
for k in fwd_band adj_gather fgp2d fwd_reduce; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:$k -s 3 -c 1 \
      -o $O/p_$k python tools/prof_kernels.py > $O/ncu_$k.log 2>&1
  ncu -i $O/p_$k.ncu-rep --page raw --csv > $O/raw_$k.csv 2>/dev/null
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:fgp3d_col -s 5 -c 1 \
    -o $O/p_fgp3d python tools/fgp3_timing.py > $O/ncu_fgp3d.log 2>&1
ncu -i $O/p_fgp3d.ncu-rep --page raw --csv > $O/raw_fgp3d.csv 2>/dev/null
PT_FGP3_PAIR=0 timeout 600 ncu --set full --import-source on --clock-control none -k regex:fgp3d_iter \
    -s 5 -c 1 -o $O/p_fgp3d_iter python tools/fgp3_timing.py > $O/ncu_fgp3d_iter.log 2>&1
ncu -i $O/p_fgp3d_iter.ncu-rep --page raw --csv > $O/raw_fgp3d_iter.csv 2>/dev/null
ls -la $O
