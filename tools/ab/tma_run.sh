O=gpurun_out
timeout 600 python -m pytest tests/test_gpu_projector.py tests/test_gpu_parity_large.py::test_full_forward_adjoint_2048 tests/test_gpu_rows.py -q -x > $O/t_tma.log 2>&1
for i in 1 2; do
 echo base >> $O/tma_times.txt; PT_LIB_OVERRIDE=$PWD/tools/ab/base.so timeout 300 python tools/kbench.py fwd >> $O/tma_times.txt 2>&1
 echo tma >> $O/tma_times.txt; timeout 300 python tools/kbench.py fwd >> $O/tma_times.txt 2>&1
 echo notma >> $O/tma_times.txt; PT_FWD_TMA=0 timeout 300 python tools/kbench.py fwd >> $O/tma_times.txt 2>&1
done
