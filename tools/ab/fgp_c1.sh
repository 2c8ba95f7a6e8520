O=gpurun_out
for cfg in "256 5 10" "256 6 10" "256 7 10" "256 8 10" "1024 7 10" "1024 7 12" "1024 7 6"; do
  set -- $cfg
  echo "big_min=$1 T=$2 t_small=$3" >> $O/fgp_c1.txt
  PT_FGP_BIG_MIN=$1 PT_FGP_T=$2 PT_FGP_T_SMALL=$3 timeout 300 python tools/kbench.py fgp 2>&1 | grep c1 >> $O/fgp_c1.txt
done
