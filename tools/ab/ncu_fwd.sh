O=gpurun_out
python tools/prof_kernels.py > $O/pk_plain.log 2>&1 && \
for c in 3 12; do
PT_FWD_CFG=$c timeout 600 ncu --set full --import-source on --clock-control none -k regex:fwd_band -s 3 -c 1 \
    -o $O/p_fwd_cfg$c python tools/prof_kernels.py > $O/ncu_fwd_$c.log 2>&1
ncu -i $O/p_fwd_cfg$c.ncu-rep --page raw --csv > $O/raw_fwd_cfg$c.csv 2>/dev/null
ncu -i $O/p_fwd_cfg$c.ncu-rep --page source --csv --print-source sass > $O/src_fwd_cfg$c.csv 2>/dev/null
done
