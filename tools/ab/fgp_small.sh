O=gpurun_out
for cfg in "256 10" "256 11" "256 12" "256 9"; do
  set -- $cfg
  echo "big_min=$1 t_small=$2" >> $O/fgp_small.txt
  PT_FGP_BIG_MIN=$1 PT_FGP_T_SMALL=$2 timeout 300 python tools/kbench.py fgp >> $O/fgp_small.txt 2>&1
done
