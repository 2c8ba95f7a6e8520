O=gpurun_out
for t in 8 5 6 7 8; do echo "T=$t" >> $O/fgp_times2.txt; PT_FGP_T=$t timeout 300 python tools/kbench.py fgp >> $O/fgp_times2.txt 2>&1; done
