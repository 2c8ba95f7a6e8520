#!/bin/bash
# Local (CPU) build of tools/ab/pdl_<mask>.so: fgp.cu / projector.cu compiled with
# -DPT_PDL_EARLY_MASK=<mask>, linked with the in-tree objects of the other sources.
set -e
cd "$(dirname "$0")/../.."
C=paper_2602_09527_b200/csrc; OBJ=paper_2602_09527_b200/_lib/obj
F="-gencode arch=compute_100a,code=sm_100a -ccbin /usr/bin/g++ -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -Xcompiler -fPIC,-fopenmp,-O3"
for m in "$@"; do
  ( nvcc $F -DPT_PDL_EARLY_MASK=$m -c $C/fgp.cu -o /tmp/fgp_$m.o &
    nvcc $F -DPT_PDL_EARLY_MASK=$m -c $C/projector.cu -o /tmp/projector_$m.o & wait )
  others=$(ls $OBJ/*.o | grep -v "/fgp.o\|/projector.o")
  nvcc -gencode arch=compute_100a,code=sm_100a -ccbin /usr/bin/g++ -shared -cudart static -o tools/ab/pdl_$m.so \
      /tmp/fgp_$m.o /tmp/projector_$m.o $others -Xcompiler -fopenmp -ldl -lpthread
  echo "built tools/ab/pdl_$m.so"
done
