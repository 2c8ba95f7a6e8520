O=gpurun_out
for f in 6 9 10 11 6; do echo "pair=$f" >> $O/fgp3_times.txt; PT_FGP3_PAIR=$f timeout 300 python tools/kbench.py fgp3 >> $O/fgp3_times.txt 2>&1; done
