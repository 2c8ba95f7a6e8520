O=gpurun_out
PT_FGP3_PAIR=6 python tools/fgp3_timing.py > $O/f3_plain.log 2>&1 && \
PT_FGP3_PAIR=6 timeout 600 ncu --set full --import-source on --clock-control none -f -k regex:fgp3d_col -s 3 -c 1 \
    -o /tmp/p_fgp3col python tools/fgp3_timing.py > $O/ncu_f3col.log 2>&1
ncu -i /tmp/p_fgp3col.ncu-rep --page raw --csv > $O/raw_fgp3col.csv 2>/dev/null
ncu -i /tmp/p_fgp3col.ncu-rep --page source --csv --print-source sass > $O/src_fgp3col.csv 2>/dev/null
