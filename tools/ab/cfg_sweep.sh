O=gpurun_out
for c in 11 12 10; do PT_FWD_CFG=$c timeout 600 python -m pytest tests/test_gpu_projector.py -q -x > $O/t_ed_$c.log 2>&1; done
for c in 3 10 11 12 13 14 15 3; do echo "cfg $c" >> $O/ed_times.txt; PT_FWD_CFG=$c timeout 300 python tools/kbench.py fwd >> $O/ed_times.txt 2>&1; done
