O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_fgp.py tests/test_gpu_rows.py -q -x > $O/t_fgp.log 2>&1
echo base >> $O/fgp_times.txt; PT_LIB_OVERRIDE=$PWD/tools/ab/base.so timeout 300 python tools/kbench.py fgp >> $O/fgp_times.txt 2>&1
for t in 8 9 10 11 12; do echo "T=$t" >> $O/fgp_times.txt; PT_FGP_T=$t timeout 300 python tools/kbench.py fgp >> $O/fgp_times.txt 2>&1; done
