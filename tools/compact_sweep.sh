#!/bin/bash
for b in 1 0; do
  MEM_NVCC_EXTRA="-DMEM_COMPACT=$b" python paper_2309_16818_b200/build.py --force > /dev/null 2>&1
  echo "compact=$b"; bash tools/qbench.sh
done
