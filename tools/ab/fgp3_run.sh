O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_fgp.py -q -x -k "3d" > $O/t_fgp3.log 2>&1
for f in 1 5 6 7 8 5; do echo "pair=$f" >> $O/fgp3_times.txt; PT_FGP3_PAIR=$f timeout 300 python tools/kbench.py fgp3 >> $O/fgp3_times.txt 2>&1; done
