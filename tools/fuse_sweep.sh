#!/bin/bash
for cfg in "2 3" "4 2" "4 3" "3 3" "1 4"; do
  set -- $cfg
  MEM_NVCC_EXTRA="-DMEM_FUSE_N=$1 -DMEM_CELLS_MINB=$2" python paper_2309_16818_b200/build.py --force > gpurun_out/fb.log 2>&1
  echo "fuse_n=$1 cells_minb=$2 spills: $(grep -c 'k_cellsILi1' gpurun_out/fb.log)"; bash tools/qbench.sh
done
