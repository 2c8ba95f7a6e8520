#!/bin/bash
# gather with staged tap pairs vs tools/ab/base.so: bits and timings
O=gpurun_out; mkdir -p $O
PT_LIB_OVERRIDE=$PWD/tools/ab/base.so python tools/gather_bits.py /tmp/gb_base.npz > $O/gb.log 2>&1
python tools/gather_bits.py /tmp/gb_new.npz >> $O/gb.log 2>&1
python -c "
import numpy as np
a=np.load('/tmp/gb_base.npz'); b=np.load('/tmp/gb_new.npz')
for k in a.files: print(k, 'bitwise' if np.array_equal(a[k], b[k]) else 'DIFF %.3g' % (np.abs(a[k]-b[k]).max()/np.abs(a[k]).max()))
" >> $O/gb.log 2>&1
for i in 1 2; do
  PT_LIB_OVERRIDE=$PWD/tools/ab/base.so timeout 600 python tools/kbench.py gather > $O/ab_base_$i.txt 2>&1
  timeout 600 python tools/kbench.py gather > $O/ab_new_$i.txt 2>&1
done
