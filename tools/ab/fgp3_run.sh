O=gpurun_out
for f in 6 5 7 8; do PT_FGP3_PAIR=$f timeout 600 python -m pytest tests/test_gpu_fgp.py -q -x -k "3d" > $O/t_fgp3_$f.log 2>&1; done
for f in 1 5 6 7 8; do echo "pair=$f" >> $O/fgp3_times.txt; PT_FGP3_PAIR=$f timeout 300 python tools/kbench.py fgp3 >> $O/fgp3_times.txt 2>&1; done
