#!/bin/bash
for mb in ${@:-3 4}; do
  MEM_NVCC_EXTRA="-DMEM_POINTS_MINB=$mb" python paper_2309_16818_b200/build.py --force > /dev/null 2>&1
  echo "points_minb=$mb"; bash tools/qbench.sh
done
