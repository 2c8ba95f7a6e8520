O=gpurun_out
timeout 1200 python -m pytest tests/test_gpu_fgp.py tests/test_gpu_solver.py -q -k "3d or zslab" > $O/t_slab.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity_large.py -q -k config3 >> $O/t_slab.log 2>&1
