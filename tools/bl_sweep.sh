#!/bin/bash
for b in 0 1; do
  MEM_NVCC_EXTRA="-DMEM_BRANCHLESS=$b" python paper_2309_16818_b200/build.py --force > /dev/null 2>&1
  echo "branchless=$b"; bash tools/qbench.sh
done
